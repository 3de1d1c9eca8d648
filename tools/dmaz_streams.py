"""DMAZ cold latency vs copy streams (groups dealt round-robin, one flag counter per stream)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2306_03622_b200 import ENGINE_DMAZ, Runtime
with Runtime(gpu_ids=[0], pool_bytes=16 << 30) as rt:
    for name in sys.argv[1:] or ["resnet50", "bert-base", "gpt2-xl"]:
        spec = synth.build_model(name)
        mid = rt.register_spec(spec, spec.build_weights(), link_code=True)
        x = spec.make_input()
        for rep in range(2):
            for streams in (1, 2, 3, 4):
                for grp in (64 << 20, 16 << 20):
                    d, sw = [], []
                    for i in range(12 if name != "gpt2-xl" else 6):
                        rt.evict(mid)
                        st = rt.invoke(mid, x, gpu=0, engine=ENGINE_DMAZ, dma_streams=streams, dma_group_bytes=grp).stats
                        d.append(st["device_ms"]); sw.append(st["swap_ms"])
                    ok = np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
                    print(f"{name:10s} streams={streams} grp={grp >> 20:3d}M p50 {np.median(d[2:]):.4f} swap {np.median(sw[2:]):.4f} copies {st['n_copies']} exact {ok}", flush=True)
        rt.unregister(mid)
