"""Cold-invoke latency of every swap engine (plain: SM, DMA; link-coded: SMZ, DMAZ) per model.

    python tools/linkcode_bench.py [models...] [--reps N] [--grp BYTES]
Prints one JSON line per (model, engine): p50/p99 device ms, swap ms, store GB/s and wire GB/s.
"""
import json
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMA, ENGINE_DMAZ, ENGINE_SM, ENGINE_SMZ, Runtime  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 20
grp = int(sys.argv[sys.argv.index("--grp") + 1]) if "--grp" in sys.argv else 0
ctas = int(sys.argv[sys.argv.index("--ctas") + 1]) if "--ctas" in sys.argv else 0
models = [a for a in args if not a.isdigit()] or ["mlp", "resnet50", "bert-base"]
with Runtime(gpu_ids=[0], pool_bytes=16 << 30) as rt:
    for name in models:
        spec = synth.build_model(name)
        w, x = spec.build_weights(), spec.make_input()
        mid = rt.register_spec(spec, w, link_code=True)
        info = rt.model_info(mid)
        rt.invoke(mid, x, gpu=0)
        warm = [rt.invoke(mid, x, gpu=0).stats["device_ms"] for _ in range(10)]
        for eng, en in ((ENGINE_SM, "sm"), (ENGINE_DMA, "dma"), (ENGINE_SMZ, "smz"), (ENGINE_DMAZ, "dmaz")):
            d, s, t, wb = [], [], [], 0
            for i in range(reps + 3):
                rt.evict(mid)
                r = rt.invoke(mid, x, gpu=0, engine=eng, dma_group_bytes=grp, copy_ctas=ctas)
                if i >= 3:
                    d.append(r.stats["device_ms"]); s.append(r.stats["swap_ms"]); t.append(r.stats["compute_tail_ms"])
                    wb = r.stats["wire_bytes"]
            ok = np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
            p50 = float(np.median(d))
            print(json.dumps({"model": name, "engine": en, "p50_ms": round(p50, 4), "p99_ms": round(float(np.max(d)), 4),
                              "swap_ms": round(float(np.median(s)), 4), "tail_ms": round(float(np.median(t)), 4),
                              "store_gbs": round(info["store_bytes"] / np.median(s) / 1e6, 2),
                              "wire_gbs": round(wb / np.median(s) / 1e6, 2), "wire_bytes": wb,
                              "resident_ms": round(float(np.median(warm)), 4), "bit_exact": ok}), flush=True)
        rt.unregister(mid)
