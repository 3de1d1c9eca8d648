import sys, time
import numpy as np
sys.path.insert(0, ".")
import synth
from paper_2306_03622_b200 import Runtime, DMA_BASELINE, NO_OVERLAP, ORDER_RANDOM, ORDER_REVERSE
CASES = [dict(), dict(order=ORDER_REVERSE), dict(order=ORDER_RANDOM, order_seed=7),
         dict(chunk_bytes=256 << 10), dict(chunk_bytes=2 << 20), dict(chunk_bytes=8 << 20),
         dict(copy_ctas=4), dict(copy_ctas=16), dict(copy_ctas=64),
         dict(flags=NO_OVERLAP), dict(flags=DMA_BASELINE)]
rt = Runtime(gpu_ids=[0], pool_bytes=8 << 30)
for name in sys.argv[1:]:
    spec = synth.build_model(name); w = spec.build_weights(); x = spec.make_input()
    mid = rt.register_spec(spec, w)
    rt.evict(mid); base = rt.invoke(mid, x, gpu=0).output.copy()
    for kw in CASES:
        rt.evict(mid)
        t = time.time()
        try:
            r = rt.invoke(mid, x, gpu=0, **kw)
            print(name, kw, f"{time.time()-t:.3f}s", "equal" if np.array_equal(r.output, base) else "DIFF", f"dev={r.stats['device_ms']:.3f}", flush=True)
        except Exception as e:
            print(name, kw, f"{time.time()-t:.3f}s", "ERROR", e, flush=True)
