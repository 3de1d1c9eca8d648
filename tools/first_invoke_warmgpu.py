"""Is the slow first cold invoke after registration the GPU clock ramp?  Warm the GPU with ~200 ms of
unrelated work (a torch matmul loop) right before the first invoke and compare."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2306_03622_b200 import Runtime
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    for trial, warm in ((0, False), (1, True), (2, False), (3, True)):
        spec = synth.build_model("bert-base", seed=200 + trial)
        mid = rt.register_spec(spec, spec.build_weights(), link_code=True)
        x = spec.make_input()
        time.sleep(5.0)  # let the GPU go idle
        if warm:
            a = torch.randn(4096, 4096, device="cuda")
            t0 = time.time()
            while time.time() - t0 < 0.2:
                a = a @ a
                a = a / a.norm()
            torch.cuda.synchronize()
        d = []
        for i in range(12):
            rt.evict(mid)
            d.append(rt.invoke(mid, x, gpu=0).stats["device_ms"])
        print(f"trial {trial} warm_gpu={warm}: first 12 cold invokes {np.round(d, 3).tolist()}", flush=True)
        rt.unregister(mid)
