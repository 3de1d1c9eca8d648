"""Small workloads for compute-sanitizer over the round-2 paths (the sanitizer serialises kernels, so libfsw
runs every invoke no-overlap): a striped DMAZ swap with virtual sources, and (FSW_MEGA=1) the persistent kernel.
    compute-sanitizer --tool memcheck python tools/sanitize_r2.py striped|mega"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMAZ, Runtime  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "striped"
spec = synth.build_model("bert-tiny")
w, x = spec.build_weights(), spec.make_input()
with Runtime(gpu_ids=[0, 0] if what == "striped" else [0], pool_bytes=1 << 30) as rt:
    mid = rt.register_spec(spec, w, link_code=True)
    if what == "striped":
        r = rt.invoke(mid, x, gpu=0, stripe=[0, 1], engine=ENGINE_DMAZ)
    else:
        r = rt.invoke(mid, x, gpu=0)
        rt.invoke(mid, x, gpu=0)
    assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    print(what, "ok", r.stats["swap_kind"], flush=True)
