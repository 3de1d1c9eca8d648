"""Small fixed workload for ncu: one cold invoke in no-overlap mode (ncu serialises kernels, so
the overlapped pipeline would deadlock under it) and N warm invokes.  Never a bench number."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth
from paper_2306_03622_b200 import ENGINE_DMA, ENGINE_DMAZ, ENGINE_SM, ENGINE_SMZ, NO_OVERLAP, Runtime

name = sys.argv[1] if len(sys.argv) > 1 else "bert-base"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
engine = {"sm": ENGINE_SM, "dma": ENGINE_DMA, "smz": ENGINE_SMZ, "dmaz": ENGINE_DMAZ}.get(sys.argv[3] if len(sys.argv) > 3 else "", 0)
coded = engine in (ENGINE_SMZ, ENGINE_DMAZ) or "coded" in sys.argv[4:]
rt = Runtime(pool_bytes=16 << 30)
spec = synth.build_model(name)
w = spec.build_weights()
x = spec.make_input()
mid = rt.register_spec(spec, w, link_code=coded)
rt.invoke(mid, x, flags=NO_OVERLAP, engine=engine if engine != ENGINE_DMAZ or "--dmaz-cold" in sys.argv else ENGINE_SMZ)
for _ in range(warm):
    rt.invoke(mid, x)
rt.close()
