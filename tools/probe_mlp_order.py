"""Probe: MLP cold latency alone vs after other models were registered in the same context
(bench r2a measured 0.2285 ms inside the extras, r1 measured 0.142 ms standalone)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_2306_03622_b200 import Runtime


def cold(rt, mid, x, n=60, warm=20, **kw):
    out = None
    ts = []
    for i in range(warm + n):
        rt.evict(mid, -1)
        r = rt.invoke(mid, x, gpu=0, **kw)
        if i >= warm:
            ts.append((r.stats["device_ms"], r.stats["swap_ms"], r.stats["wire_bytes"]))
    a = np.array(ts)
    return {"p50": float(np.median(a[:, 0])), "swap": float(np.median(a[:, 1])), "wire_gbs": float(a[0, 2] / np.median(a[:, 1]) / 1e6)}


def meminfo():
    d = {}
    for l in open("/proc/meminfo"):
        k, v = l.split(":", 1)
        if k in ("AnonHugePages", "HugePages_Total", "MemFree", "MemAvailable"):
            d[k] = v.strip()
    return d


print("thp", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip(), meminfo(), flush=True)
rt = Runtime(gpu_ids=[0], pool_bytes=16 << 30)
mspec = synth.build_model("mlp")
mw, mx = mspec.build_weights(), mspec.make_input()
m1 = rt.register_spec(mspec, mw, link_code=True)
print("mlp alone", cold(rt, m1, mx), meminfo(), flush=True)
bspec = synth.build_model("bert-base")
b = rt.register_spec(bspec, bspec.build_weights(), link_code=True)
bx = bspec.make_input()
print("bert", cold(rt, b, bx, n=20, warm=5), flush=True)
print("mlp after bert registered (same store)", cold(rt, m1, mx), flush=True)
m2 = rt.register_spec(mspec, mw, link_code=True)
print("mlp re-registered after bert", cold(rt, m2, mx), meminfo(), flush=True)
rt.unregister(b)
m3 = rt.register_spec(mspec, mw, link_code=True)
print("mlp re-registered after bert unregistered", cold(rt, m3, mx), flush=True)
for c in (16, 32, 48, 64):
    print("mlp ctas", c, cold(rt, m1, mx, copy_ctas=c), flush=True)
