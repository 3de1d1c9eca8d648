"""A few cold striped invokes of one model over N pool GPUs (for ncu's NVLink / PCIe counters on a
multi-GPU box: tools/ncu_nvlink.sh).  On a 1-GPU box the pool lists device 0 N times (virtual sources:
same protocol, NVLink counters stay 0).

    python tools/striped_once.py [--gpus N] [--model gpt2-xl] [--engine 3|4] [--reps 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import ENGINE_DMAZ, Runtime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--model", default="gpt2-xl")
    ap.add_argument("--engine", type=int, default=ENGINE_DMAZ)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--pool-gb", type=int, default=8)
    args = ap.parse_args()
    import torch
    ndev = max(1, torch.cuda.device_count())
    ids = [i % ndev for i in range(args.gpus)]
    spec = synth.build_model(args.model)
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=ids, pool_bytes=args.pool_gb << 30, stripe_min_bytes=1) as rt:
        mid = rt.register_spec(spec, w, link_code=True)
        del w
        for _ in range(args.reps):
            rt.evict(mid)
            r = rt.invoke(mid, x, gpu=0, stripe=list(range(args.gpus)), engine=args.engine)
            st = r.stats
            print(json.dumps({"devices": ids, "device_ms": round(st["device_ms"], 3), "swap_ms": round(st["swap_ms"], 3),
                              "wire_bytes": st["wire_bytes"], "n_sources": st["n_sources"], "engine": st["engine"],
                              "wire_gbs": round(st["wire_bytes"] / (st["swap_ms"] * 1e6), 2)}), flush=True)
        assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid)), "striped swap bytes differ"


if __name__ == "__main__":
    main()
