"""Swap-engine sweep on the GPU box: SM swap kernel (piece size, CTAs) vs copy-engine DMA (group
size, copy streams), cold invoke p50 and swap GB/s per model.  Exploration tool, not the bench.

    python tools/engine_sweep.py bert-base resnet50 mlp [gpt2-xl]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2306_03622_b200 import DMA_BASELINE, ENGINE_DMA, ENGINE_SM, Runtime  # noqa: E402

names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["bert-base", "resnet50", "mlp"]
reps = 9
rt = Runtime(gpu_ids=[0], pool_bytes=24 << 30)
res = {}
for n in names:
    spec = synth.build_model(n)
    w = spec.build_weights()
    x = spec.make_input()
    mid = rt.register_spec(spec, w)
    B = rt.model_info(mid)["store_bytes"]

    def run(**kw):
        st = []
        for i in range(reps + 2):
            rt.evict(mid)
            s = rt.invoke(mid, x, gpu=0, **kw).stats
            if i >= 2:
                st.append(s)
        d = float(np.median([s["device_ms"] for s in st]))
        sw = float(np.median([s["swap_ms"] for s in st]))
        tail = float(np.median([s["compute_tail_ms"] for s in st]))
        return {"p50": round(d, 4), "swap": round(sw, 4), "gbs": round(B / sw / 1e6, 2), "tail": round(tail, 4),
                "copies": st[0]["n_copies"]}

    rows = {}
    for chunk in (16 << 10, 32 << 10, 64 << 10, 256 << 10):
        for ctas in (8, 16, 32):
            rows[f"sm chunk={chunk >> 10}K ctas={ctas}"] = run(engine=ENGINE_SM, chunk_bytes=chunk, copy_ctas=ctas)
    rows["paper dma 2MB x1"] = run(flags=DMA_BASELINE)
    for grp in (4, 8, 16, 32, 64):
        for streams in (1, 2):
            rows[f"dma grp={grp}M streams={streams}"] = run(engine=ENGINE_DMA, dma_group_bytes=grp << 20,
                                                           dma_streams=streams)
    warm = [rt.invoke(mid, x, gpu=0).stats["device_ms"] for _ in range(reps)]
    print(f"== {n}: store {B} B, resident p50 {np.median(warm):.4f} ms", flush=True)
    for k, v in sorted(rows.items(), key=lambda kv: kv[1]["p50"]):
        print(f"   {k:28s} p50 {v['p50']:8.4f} ms  swap {v['swap']:8.4f} ms  {v['gbs']:6.2f} GB/s  tail {v['tail']:.4f}  copies {v['copies']}", flush=True)
    res[n] = {"store_bytes": B, "resident_p50": float(np.median(warm)), "rows": rows}
    rt.unregister(mid)
rt.close()
json.dump(res, open("gpurun_out/engine_sweep.json", "w"), indent=1)
