"""The analogue of the paper's tab:eval_remote_swap on one B200: per model the
resident latency (~ "Remote Async"), the non-pipelined cold invoke (swap, then run: FSW_NO_OVERLAP,
~ "Non-pipeline"), and the pipelined cold invoke (~ "Pipeline PCIe") with the plain store and with
the link-coded store; the paper's V100 numbers beside them (different hardware, fp32: context).

    python tools/paper_table.py [--reps 20] [models...]
"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMA, NO_OVERLAP, Runtime  # noqa: E402

PAPER = {  # Remote Async, Non-pipeline, Pipeline PCIe (ms, 4x V100, fp32)
    "resnet50": (9, 23, 13), "resnet101": (14, 35, 22), "resnet152": (19, 45, 29), "bert-large": (45, 190, 149),
}
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 20
names = [a for a in sys.argv[1:] if not a.startswith("--") and not a.isdigit()] or list(PAPER)
rows = []
with Runtime(gpu_ids=[0], pool_bytes=16 << 30) as rt:
    for name in names:
        spec = synth.build_model(name)
        w, x = spec.build_weights(), spec.make_input()
        plain = rt.register_spec(spec, w)
        coded = rt.register_spec(spec, w, link_code=True)

        def med(fn, warm_s=0.5):  # untimed warm-up by time (the first cold invokes after registration run slower)
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < warm_s:
                fn()
            v = [fn() for _ in range(reps)]
            return round(float(np.median(v)), 4)

        def cold(mid, **kw):
            rt.evict(mid)
            return rt.invoke(mid, x, gpu=0, **kw).stats["device_ms"]

        rt.invoke(plain, x, gpu=0)
        row = {"model": name, "store_mb": round(rt.model_info(plain)["store_bytes"] / 1e6, 1),
               "resident_ms": med(lambda: rt.invoke(plain, x, gpu=0).stats["device_ms"]),
               "non_pipelined_ms": med(lambda: cold(plain, engine=ENGINE_DMA, flags=NO_OVERLAP)),
               "pipelined_plain_ms": med(lambda: cold(plain)),
               "pipelined_coded_ms": med(lambda: cold(coded)),
               "paper_v100_resident_nonpipe_pipe_ms": PAPER.get(name)}
        print(json.dumps(row), flush=True)
        rows.append(row)
        rt.unregister(plain)
        rt.unregister(coded)
