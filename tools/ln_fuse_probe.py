"""Folded LayerNorm (FSW_LN_FUSE, read once per process): output vs the oracle, resident and cold p50, kernels per
invoke, for the transformer models.  Run once with FSW_LN_FUSE=0 and once with =1.
    FSW_LN_FUSE=1 python tools/ln_fuse_probe.py [bert-tiny bert-base ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402

names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["bert-tiny", "bert-base", "gpt2-tiny"]
fuse = os.environ.get("FSW_LN_FUSE", "0")
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    for name in names:
        spec = synth.build_model(name)
        w, x = spec.build_weights(), spec.make_input()
        mid = rt.register_spec(spec, w, link_code=name.endswith("base"))
        r = rt.invoke(mid, x, gpu=0)
        ref = oracle.output(spec, w, x).reshape(-1)
        got = r.output.astype(np.float64).reshape(-1)
        err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
        res = []
        for _ in range(200):
            res.append(rt.invoke(mid, x, gpu=0).stats["device_ms"])
        cold = []
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.5:
            rt.evict(mid)
            rt.invoke(mid, x, gpu=0)
        for _ in range(30):
            rt.evict(mid)
            cold.append(rt.invoke(mid, x, gpu=0).stats["device_ms"])
        r2 = rt.invoke(mid, x, gpu=0)
        same = bool(np.array_equal(r2.output, r.output))
        print(f"FSW_LN_FUSE={fuse} {name}: rel err {err:.3e}, resident p50 {np.median(res):.4f} ms, cold p50 "
              f"{np.median(cold):.4f} ms, kernels/invoke {r.stats['n_kernels']}, warm == cold {same}", flush=True)
        rt.unregister(mid)
