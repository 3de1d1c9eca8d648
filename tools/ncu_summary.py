"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel totals and
the share of each kernel family, optionally restricted to the last N launches (one invoke)."""
import csv, sys, collections, re

def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        rows.append((int(r["ID"]), r["Kernel Name"], ns))
    return rows

def family(name):
    m = re.match(r"(?:void )?(?:fsw::)?(k_\w+)", name)
    return m.group(1) if m else name[:40]

if __name__ == "__main__":
    path = sys.argv[1]
    rows = load(path)
    start = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    end = int(sys.argv[3]) if len(sys.argv) > 3 else len(rows)
    sel = rows[start:end]
    tot = sum(r[2] for r in sel)
    fam = collections.defaultdict(lambda: [0, 0.0])
    for _, n, ns in sel:
        f = fam[family(n)]; f[0] += 1; f[1] += ns
    print(f"launches {start}..{end} of {len(rows)}: {len(sel)} kernels, sum {tot/1e3:.1f} us")
    for k, (c, ns) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:28s} n={c:4d} sum={ns/1e3:9.1f} us  mean={ns/c/1e3:8.2f} us  share={ns/tot*100:5.1f}%")
