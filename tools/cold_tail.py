"""Tail of the cold-invoke latency distribution (p50 / p90 / p99 / max over N cold invokes) per engine setting.
    python tools/cold_tail.py [model] [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert-base"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
spec = synth.build_model(name)
w, x = spec.build_weights(), spec.make_input()
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FSW_")) or "default"
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    mid = rt.register_spec(spec, w, link_code=True)
    for _ in range(20):
        rt.evict(mid)
        rt.invoke(mid, x, gpu=0)
    d, sw = [], []
    for _ in range(n):
        rt.evict(mid)
        st = rt.invoke(mid, x, gpu=0).stats
        d.append(st["device_ms"])
        sw.append(st["swap_ms"])
    d = np.array(d)
    q = lambda p: float(np.percentile(d, p))
    slow = np.argsort(d)[-5:]
    print(f"[{tag}] {name} cold x{n}: p50 {q(50):.4f} p90 {q(90):.4f} p99 {q(99):.4f} max {d.max():.4f} ms; "
          f"slowest at steps {sorted(slow.tolist())}, their swap_ms {[round(sw[i], 3) for i in sorted(slow.tolist())]}", flush=True)
