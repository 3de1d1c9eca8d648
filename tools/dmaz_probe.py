"""DMAZ decode capacity: cold BERT-base invokes for decoder kernel x CTA count, overlapped and serial
(NO_OVERLAP: every copy group first, then the decode, then the layers; decode ms = device − copy − resident).

    FSW_SWAPZ_REGS=1 python tools/dmaz_probe.py   # the register decoder instead of the TMA ring
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMAZ, ENGINE_SMZ, NO_OVERLAP, Runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert-base"
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    spec = synth.build_model(name)
    w, x = spec.build_weights(), spec.make_input()
    mid = rt.register_spec(spec, w, link_code=True)
    info = rt.model_info(mid)
    rt.invoke(mid, x, gpu=0)
    res = float(np.median([rt.invoke(mid, x, gpu=0).stats["device_ms"] for _ in range(10)]))
    for eng, en in ((ENGINE_DMAZ, "dmaz"), (ENGINE_SMZ, "smz")):
        for ctas in (32, 48, 64, 96):
            for flags, fn in ((0, "overlap"), (NO_OVERLAP, "serial")):
                d = []
                for i in range(13):
                    rt.evict(mid)
                    r = rt.invoke(mid, x, gpu=0, engine=eng, copy_ctas=ctas, flags=flags)
                    if i >= 3:
                        d.append(r.stats["device_ms"])
                p50 = float(np.median(d))
                out = {"engine": en, "regs": bool(os.environ.get("FSW_SWAPZ_REGS")), "ctas": ctas, "mode": fn,
                       "p50_ms": round(p50, 4), "resident_ms": round(res, 4)}
                if fn == "serial" and en == "dmaz":
                    copy = info["coded_bytes"] / 55.4e6
                    out["decode_ms_est"] = round(p50 - res - copy, 4)
                    out["decode_store_gbs_est"] = round(info["store_bytes"] / max(1e-6, p50 - res - copy) / 1e6, 1)
                print(json.dumps(out), flush=True)
    assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
