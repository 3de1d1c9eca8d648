"""Small workloads for compute-sanitizer over the round-2 paths (the sanitizer serialises kernels, so libfsw
runs every invoke no-overlap): a striped DMAZ swap with virtual sources, (FSW_MEGA=1) the persistent kernel, and
`ws`: entropy-coded pieces (v5) through SMZ and DMAZ, every linear on k_gemm_ws (split-K push reduction), and
(FSW_ATTN_TC=1) the tcgen05 attention.
    compute-sanitizer --tool memcheck python tools/sanitize_r2.py striped|mega|ws"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMAZ, ENGINE_SMZ, Runtime  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "striped"
if what == "ws":
    os.environ["FSW_LINK_HUFF"] = "1"  # read at registration (the store is below the 32-MiB threshold)
spec = synth.build_model("bert-tiny")
w, x = spec.build_weights(), spec.make_input()
with Runtime(gpu_ids=[0, 0] if what == "striped" else [0], pool_bytes=1 << 30) as rt:
    mid = rt.register_spec(spec, w, link_code=True)
    if what == "striped":
        r = rt.invoke(mid, x, gpu=0, stripe=[0, 1], engine=ENGINE_DMAZ)
    elif what == "ws":
        assert rt.coded_code(mid).any()
        for eng in (ENGINE_SMZ, ENGINE_DMAZ):
            rt.evict(mid)
            r = rt.invoke(mid, x, gpu=0, engine=eng)
            assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
        rt.invoke(mid, x, gpu=0)
    else:
        r = rt.invoke(mid, x, gpu=0)
        rt.invoke(mid, x, gpu=0)
    assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    print(what, "ok", r.stats["swap_kind"], flush=True)
