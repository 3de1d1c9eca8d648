"""How a copy group is published (FSW_DMA_FLAG, read once per process): cold p50 of the copy-engine engines.
    FSW_DMA_FLAG=1 python tools/dma_flag_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMA, ENGINE_DMAZ, ENGINE_DMAZT, ENGINE_SMZ, Runtime  # noqa: E402

mode = os.environ.get("FSW_DMA_FLAG", "0")


def cold(rt, mid, x, reps=40, **kw):
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.4:
        rt.evict(mid)
        rt.invoke(mid, x, gpu=0, **kw)
    v = []
    for _ in range(reps):
        rt.evict(mid)
        v.append(rt.invoke(mid, x, gpu=0, **kw).stats["device_ms"])
    return float(np.median(v))


with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    for name in ("resnet50", "bert-base"):
        spec = synth.build_model(name)
        w, x = spec.build_weights(), spec.make_input()
        z = rt.register_spec(spec, w, link_code=True)
        p = rt.register_spec(spec, w)
        row = {"dmazt": cold(rt, z, x, engine=ENGINE_DMAZT), "dmaz": cold(rt, z, x, engine=ENGINE_DMAZ),
               "smz": cold(rt, z, x, engine=ENGINE_SMZ), "dma": cold(rt, p, x, engine=ENGINE_DMA)}
        print(f"FSW_DMA_FLAG={mode} {name}: " + " ".join(f"{k} {v:.4f}" for k, v in row.items()), flush=True)
        rt.unregister(z)
        rt.unregister(p)
