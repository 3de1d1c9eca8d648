"""Extract the judged counters of an ncu --set full report into a small text/JSON summary.

    python tools/ncu_extract.py gpurun_out/prof_swap.ncu-rep [out.json]

Reads `ncu -i <rep> --page raw --csv` (no GPU needed) and keeps, per profiled launch: duration,
grid, DRAM/PCIe/sysmem traffic, tensor-pipe activity and occupancy."""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "pcie__read_bytes.sum", "pcie__write_bytes.sum", "pcie__read_bytes.sum.per_second",
    "syslts__t_sectors_aperture_sysmem_op_read.sum", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "Kbyte/block": 1e3, "byte/block": 1, "Gbyte/s": 1e9, "Mbyte/s": 1e6, "Tbyte/s": 1e12}


def extract(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")][:80], "id": r[head.index("ID")]}
        for k in KEEP:
            if k in head:
                i = head.index(k)
                v = r[i].replace(",", "")
                try:
                    d[k] = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    d[k] = v
        out.append(d)
    return out


if __name__ == "__main__":
    res = extract(sys.argv[1])
    s = json.dumps(res, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s + "\n")
    print(s)
