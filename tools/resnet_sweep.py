"""ResNet-50 cold invoke: link format (v4 / v5) x engine (SMZ / DMAZ / DMAZT) x decode CTAs x copy-group size.
Which combination brings the 51-MB store closest to its coded-byte roofline (1.29x, target 1.2x)?
    python tools/resnet_sweep.py [model] [--quick]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMAZ, ENGINE_DMAZT, ENGINE_SMZ, Runtime  # noqa: E402

name = next((a for a in sys.argv[1:] if not a.startswith("--")), "resnet50")
spec = synth.build_model(name)
w, x = spec.build_weights(), spec.make_input()


def cold(rt, mid, reps=60, **kw):
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.4:
        rt.evict(mid)
        rt.invoke(mid, x, gpu=0, **kw)
    v, wire = [], 0
    for _ in range(reps):
        rt.evict(mid)
        r = rt.invoke(mid, x, gpu=0, **kw)
        v.append(r.stats["device_ms"])
        wire = r.stats["wire_bytes"]
    return float(np.median(v)), wire


with Runtime(gpu_ids=[0], pool_bytes=4 << 30) as rt:
    mids = {}
    for fmt, hv in (("v4", "0"), ("v5", "1")):
        os.environ["FSW_LINK_HUFF"] = hv
        mids[fmt] = rt.register_spec(spec, w, link_code=True)
    del os.environ["FSW_LINK_HUFF"]
    for fmt, mid in mids.items():
        ms, wire = cold(rt, mid, engine=ENGINE_SMZ)
        print(f"{name} {fmt} smz default            {ms:.4f} ms  wire {wire/1e6:.2f} MB  {wire/ms/1e6:.1f} GB/s", flush=True)
        for ctas in (0, 64, 96, 128):
            for grp in (4 << 20, 8 << 20, 16 << 20, 64 << 20):
                for eng, en in ((ENGINE_DMAZ, "dmaz"), (ENGINE_DMAZT, "dmazt")):
                    try:
                        ms, wire = cold(rt, mid, engine=eng, copy_ctas=ctas, dma_group_bytes=grp)
                    except Exception as e:  # noqa: BLE001
                        print(f"{name} {fmt} {en} ctas={ctas} grp={grp >> 20} failed: {e}", flush=True)
                        continue
                    print(f"{name} {fmt} {en:5s} ctas={ctas:3d} grp={grp >> 20:2d}MiB {ms:.4f} ms  {wire/ms/1e6:.1f} GB/s", flush=True)
