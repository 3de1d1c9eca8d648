# Per-source NVLink and PCIe bytes of a striped cold invoke, for
# the first multi-GPU box:  bash tools/ncu_nvlink.sh [N] [engine 3=SMZ|4=DMAZ] [model]
# ncu serialises kernels, so libfsw runs the invoke no-overlap (profiler-safe mode): every source's swap /
# decode kernel is captured alone.  nvltx__bytes at a source = bytes it stored into the target over NVLink;
# nvlrx__bytes at the target = what it received; pcie__read_bytes = the source's own host-link reads (SMZ;
# with DMAZ the copy engine reads outside any kernel, so compare the staged run bytes instead).
N=${1:-2}; ENG=${2:-3}; MODEL=${3:-gpt2-xl}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_write.sum \
    -k regex:k_swap --csv --log-file gpurun_out/ncu_nvlink_n${N}_e${ENG}.csv \
    python tools/striped_once.py --gpus $N --engine $ENG --model $MODEL --reps 1
python - "$N" "$ENG" <<'PY'
import csv, sys, collections
n, e = sys.argv[1], sys.argv[2]
rows = list(csv.DictReader(l for l in open(f"gpurun_out/ncu_nvlink_n{n}_e{e}.csv") if l.startswith('"')))
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows:
    try:
        v = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    agg[(r.get("Device", r.get("device", "?")), r["Kernel Name"][:40])][r["Metric Name"]] += v
for k, d in sorted(agg.items()):
    print(k, {m: round(v / (1e9 if "bytes" in m else 1e6), 4) for m, v in d.items()}, "(GB / ms)")
PY
