"""Quick check of the persistent transformer kernel: cold and resident invokes vs the oracle, resident time.
    python tools/mega_quick.py [model ...]"""
import os
import sys
import time

os.environ.setdefault("FSW_MEGA", "1")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402

names = sys.argv[1:] or ["bert-tiny", "gpt2-tiny", "bert-base", "gpt2-2L"]
with Runtime(gpu_ids=[0], pool_bytes=4 << 30) as rt:
    for name in names:
        spec = synth.build_model(name)
        w, x = spec.build_weights(), spec.make_input()
        mid = rt.register_spec(spec, w, link_code=True)
        ref = oracle.output(spec, w, x).reshape(-1)
        t0 = time.time()
        r = rt.invoke(mid, x, gpu=0)
        cold = r.output.astype(np.float64).reshape(-1)
        err = float(np.max(np.abs(cold - ref)) / np.max(np.abs(ref)))
        ok_bytes = np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
        warm = [rt.invoke(mid, x, gpu=0) for _ in range(30)]
        same = all(np.array_equal(wv.output, r.output) for wv in warm)
        res = sorted(wv.stats["device_ms"] for wv in warm)[15]
        colds = []
        for _ in range(10):
            rt.evict(mid)
            colds.append(rt.invoke(mid, x, gpu=0).stats["device_ms"])
        print(f"{name}: rel err {err:.3e} bytes_ok {ok_bytes} warm==cold {same} resident p50 {res:.4f} ms "
              f"cold p50 {sorted(colds)[5]:.4f} ms kernels/invoke {r.stats['n_kernels']}", flush=True)
        rt.unregister(mid)
