"""Quick A/B of the weight-stationary GEMM (k_gemm_ws): cold and resident invokes vs the oracle, resident and
cold p50.  Run once per setting (env is read once per process):
    FSW_GEMM_WS=1 python tools/ws_quick.py [model ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402

names = sys.argv[1:] or ["bert-tiny", "gpt2-tiny", "bert-base"]
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FSW_")) or "default"
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    for name in names:
        spec = synth.build_model(name)
        w, x = spec.build_weights(), spec.make_input()
        mid = rt.register_spec(spec, w, link_code=True)
        ref = oracle.output(spec, w, x).reshape(-1) if name != "gpt2-xl" else None
        r = rt.invoke(mid, x, gpu=0)
        err = float("nan")
        if ref is not None:
            cold = r.output.astype(np.float64).reshape(-1)
            err = float(np.max(np.abs(cold - ref)) / np.max(np.abs(ref)))
        warm = [rt.invoke(mid, x, gpu=0) for _ in range(40)]
        same = all(np.array_equal(wv.output, r.output) for wv in warm)
        res = sorted(wv.stats["device_ms"] for wv in warm)[20]
        colds = []
        for _ in range(10):
            rt.evict(mid)
            colds.append(rt.invoke(mid, x, gpu=0).stats["device_ms"])
        print(f"[{tag}] {name}: rel err {err:.3e} warm==cold {same} resident p50 {res:.4f} ms "
              f"cold p50 {sorted(colds)[5]:.4f} ms kernels/invoke {r.stats['n_kernels']}", flush=True)
        rt.unregister(mid)
