"""Stability of cold-invoke latency per engine over time (SM-issued zero-copy reads vs the copy
engine), with nvidia-smi SM clocks sampled per batch."""
import os, subprocess, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2306_03622_b200 import ENGINE_DMAZ, ENGINE_SM, ENGINE_SMZ, ENGINE_DMA, Runtime

def clk():
    return subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.mem,power.draw,pstate", "--format=csv,noheader"],
                          capture_output=True, text=True).stdout.strip()

with Runtime(gpu_ids=[0], pool_bytes=16 << 30) as rt:
    spec = synth.build_model("resnet50")
    mid = rt.register_spec(spec, spec.build_weights(), link_code=True)
    x = spec.make_input()
    t_end = time.time() + float(sys.argv[1] if len(sys.argv) > 1 else 20)
    batch = 0
    while time.time() < t_end:
        for eng, en in ((ENGINE_SMZ, "smz"), (ENGINE_DMAZ, "dmaz"), (ENGINE_SM, "sm"), (ENGINE_DMA, "dma")):
            dev = []
            for i in range(20):
                rt.evict(mid)
                dev.append(rt.invoke(mid, x, gpu=0, engine=eng).stats["device_ms"])
            print(f"t={batch:3d} {en:5s} p50 {np.median(dev):.4f} min {min(dev):.4f} max {max(dev):.4f}  [{clk()}]", flush=True)
        batch += 1
