"""Concurrent-swap interference on one host link (the analogue of the paper's
Table 3): cold invoke latency of model X alone, and while model Y cold-swaps
at the same time over the SAME PCIe link.  The paper's GPU pairs shared a PCIe switch;
here two pool GPUs are mapped onto one B200 (`gpu_ids=[0, 0]`), so both swaps share its Gen5 x16
link (and its SMs).  Prints the slowdown matrix.

    python tools/interference.py [--reps 9] [--models mlp,resnet50,bert-base,gpt2-2L]
"""
import argparse
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--models", default="mlp,resnet50,bert-base,gpt2-2L")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "interference.json"))
    ap.add_argument("--link-code", action="store_true", help="register the models link-coded (SMZ / DMAZ engines)")
    args = ap.parse_args()
    names = args.models.split(",")
    rt = Runtime(gpu_ids=[0, 0], pool_bytes=3 << 30)
    mids, xs = {}, {}
    for n in names:
        sp = synth.build_model(n)
        mids[n] = rt.register_spec(sp, sp.build_weights(), link_code=args.link_code)
        xs[n] = sp.make_input()

    def cold(n, gpu):
        rt.evict(mids[n])
        return rt.invoke(mids[n], xs[n], gpu=gpu).stats["device_ms"]

    alone = {}
    for n in names:
        for _ in range(2):
            cold(n, 0)
        alone[n] = float(np.median([cold(n, 0) for _ in range(args.reps)]))
    res = {}
    for x in names:
        for y in names:
            if x == y:
                continue
            lat = []
            for _ in range(args.reps + 1):
                rt.evict(mids[x])
                rt.evict(mids[y])
                bar = threading.Barrier(2)
                out = {}

                def run(n, gpu):
                    bar.wait()
                    out[n] = rt.invoke(mids[n], xs[n], gpu=gpu).stats["device_ms"]

                ty = threading.Thread(target=run, args=(y, 1))
                ty.start()
                run(x, 0)
                ty.join()
                lat.append(out[x])
            res[f"{x}|{y}"] = {"ms": round(float(np.median(lat[1:])), 4),
                               "slowdown": round(float(np.median(lat[1:])) / alone[x], 3)}
    summary = {"alone_ms": {k: round(v, 4) for k, v in alone.items()}, "with": res,
               "setup": "two pool GPUs on one B200: both cold swaps share one PCIe Gen5 x16 link and the SMs"}
    print(json.dumps(summary, indent=1), flush=True)
    json.dump(summary, open(args.out, "w"), indent=1)
    rt.close()


if __name__ == "__main__":
    main()
