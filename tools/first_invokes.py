"""Cold-invoke latency of the first invokes after registration, one by one (does a freshly pinned
store read slower until warmed?)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2306_03622_b200 import ENGINE_DMAZ, ENGINE_SMZ, ENGINE_DMA, Runtime
eng = {"smz": ENGINE_SMZ, "dmaz": ENGINE_DMAZ, "dma": ENGINE_DMA}[sys.argv[1] if len(sys.argv) > 1 else "smz"]
name = sys.argv[2] if len(sys.argv) > 2 else "resnet50"
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    for trial in range(2):
        spec = synth.build_model(name, seed=100 + trial)
        t = time.time(); mid = rt.register_spec(spec, spec.build_weights(), link_code=eng != ENGINE_DMA); treg = time.time() - t
        x = spec.make_input()
        d = []
        for i in range(40):
            rt.evict(mid)
            d.append(rt.invoke(mid, x, gpu=0, engine=eng).stats["device_ms"])
        print(f"{sys.argv[1:]} trial {trial} reg {treg:.2f}s first10 {np.round(d[:10], 3).tolist()} median(20:) {np.median(d[20:]):.4f}", flush=True)
        rt.unregister(mid)
