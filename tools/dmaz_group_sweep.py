"""DMAZT (format v5) copy-group cap x tail taper x head ramp: cold p50 (BERT-base; GPT-2-XL with --gpt).
    FSW_DMAZ_TAPER / FSW_DMAZ_RAMP from the environment; group caps swept here."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402

tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FSW_")) or "default"
for name in (["gpt2-xl"] if "--gpt" in sys.argv else ["bert-base"]):
    spec = synth.build_model(name)
    w, x = spec.build_weights(), spec.make_input()
    reps = 10 if name == "gpt2-xl" else 60
    with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
        mid = rt.register_spec(spec, w, link_code=True)
        for grp in (32 << 20, 64 << 20, 128 << 20, 256 << 20):
            for _ in range(5):
                rt.evict(mid)
                rt.invoke(mid, x, gpu=0, dma_group_bytes=grp)
            d = []
            for _ in range(reps):
                rt.evict(mid)
                d.append(rt.invoke(mid, x, gpu=0, dma_group_bytes=grp).stats["device_ms"])
            print(f"[{tag}] {name} grp {grp >> 20} MiB: cold p50 {np.median(d):.4f} ms", flush=True)
