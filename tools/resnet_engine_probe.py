"""ResNet-50 cold invoke with SMZ vs DMAZ (group-size / ramp / taper variants): which engine wins a 51-MB store.
    python tools/resnet_engine_probe.py [model]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMAZ, ENGINE_DMAZT, ENGINE_SMZ, Runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
spec = synth.build_model(name)
w, x = spec.build_weights(), spec.make_input()


def cold(rt, mid, reps=60, **kw):
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.5:
        rt.evict(mid)
        rt.invoke(mid, x, gpu=0, **kw)
    v = []
    for _ in range(reps):
        rt.evict(mid)
        v.append(rt.invoke(mid, x, gpu=0, **kw).stats["device_ms"])
    return float(np.median(v))


with Runtime(gpu_ids=[0], pool_bytes=4 << 30) as rt:
    mid = rt.register_spec(spec, w, link_code=True)
    print(name, "smz", round(cold(rt, mid, engine=ENGINE_SMZ), 4), flush=True)
    print(name, "dmazt", os.environ.get("FSW_DMAZT_TAIL_MB", "7"), round(cold(rt, mid, engine=ENGINE_DMAZT), 4), flush=True)
    for grp in (4 << 20, 8 << 20, 16 << 20, 64 << 20) if "--dmaz" in sys.argv else ():
        print(name, "dmaz grp", grp >> 20, "MiB", round(cold(rt, mid, engine=ENGINE_DMAZ, dma_group_bytes=grp), 4), flush=True)
