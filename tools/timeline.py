"""Device timeline of one cold invoke and one resident invoke (FSW_TRACE; DESIGN.md §5 "Overlap
timeline"): per layer, when its swap pieces were released (first / last), when its kernel passed the
weight wait, and when its last CTA exited — the evidence that "the transmission of subsequent layers
[overlaps] with the computation of previous layers".  nsys is not in this image, so
the timeline comes from %globaltimer stamps the kernels write themselves.

    python -m paper_2306_03622_b200.build --trace; python tools/timeline.py [--model bert-base] [--engine 0] [--out gpurun_out/timeline_bert.txt]
"""
import argparse
import os
import sys

os.environ.setdefault("FSW_TRACE", "1")
os.environ.setdefault("FSW_LIB", "libfsw_trace.so")  # the build with the stamps compiled into the kernels
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402

OPS = {1: "embed", 2: "layernorm", 3: "linear", 4: "attention", 5: "conv2d", 6: "maxpool", 7: "avgpool"}


def table(spec, rt, mid, tr, ti, title, out):
    t0 = min([v for v in tr[:, 0] if v] + [v for v in tr[:, 3] if v] + ([int(ti[0])] if ti[0] else []))
    us = lambda v: (int(v) - t0) / 1e3 if v else float("nan")
    out.append(f"== {title}: t = 0 at the first event; times in us ==")
    out.append(f"{'layer':>5} {'op':<10} {'name':<28} {'MB':>7} {'rel.first':>9} {'rel.last':>9} {'entry':>9} "
               f"{'wait.done':>9} {'exit':>9}")
    seen = set()
    for li, l in enumerate(spec.layers):
        mb = sum(spec.tensors[r].nbytes for r in l.refs if r not in seen) / 1e6
        seen.update(l.refs)
        e = tr[li]
        out.append(f"{li:>5} {OPS.get(int(l.op), '?'):<10} {l.name[:28]:<28} {mb:>7.2f} {us(e[3]):>9.1f} {us(e[4]):>9.1f} "
                   f"{us(e[0]):>9.1f} {us(e[1]):>9.1f} {us(e[2]):>9.1f}")
    ends = [int(v) for v in tr[:, 2] if v]
    rel = [int(v) for v in tr[:, 4] if v]
    total = (max(ends) - t0) / 1e3
    out.append(f"last kernel exit {total:.1f} us" + (f"; last piece released {(max(rel) - t0) / 1e3:.1f} us; "
                                                     f"compute after the last byte {(max(ends) - max(rel)) / 1e3:.1f} us"
                                                     if rel else ""))
    return total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="bert-base")
    ap.add_argument("--engine", type=int, default=0, help="0 auto (coded: DMAZ / SMZ), 1 SM, 2 DMA, 3 SMZ, 4 DMAZ")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--phases", action="store_true", help="resident GEMM phases (fields 5-7: last pdl_wait return, "
                    "last MMA completion, last epilogue start)")
    args = ap.parse_args()
    spec = synth.build_model(args.model)
    w, x = spec.build_weights(), spec.make_input()
    out = []
    with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
        mid = rt.register_spec(spec, w, link_code=True)
        for _ in range(args.reps):  # warm-up: clocks, first-invoke effects
            rt.evict(mid)
            r = rt.invoke(mid, x, gpu=0, engine=args.engine)
        st = r.stats
        out.append(f"{args.model}: cold invoke device {st['device_ms']:.3f} ms, swap {st['swap_ms']:.3f} ms, engine "
                   f"{st['engine']}, wire bytes {st['wire_bytes']}")
        tr, ti = rt.trace(mid)
        table(spec, rt, mid, tr, ti, f"cold invoke ({args.model}, engine {st['engine']})", out)
        for _ in range(args.reps):
            r = rt.invoke(mid, x, gpu=0)
        out.append(f"\n{args.model}: resident invoke device {r.stats['device_ms']:.3f} ms")
        tr, ti = rt.trace(mid)
        table(spec, rt, mid, tr, ti, f"resident invoke ({args.model})", out)
        if args.phases:
            t0 = min(int(v) for v in tr[:, 0] if v)
            us = lambda v: (int(v) - t0) / 1e3 if v else float("nan")
            out.append(f"{'layer':>5} {'name':<22} {'entry':>8} {'wait.w':>8} {'pdl.wait':>8} {'mma.done':>8} {'staged':>8} {'epi':>8} "
                       f"{'loaded':>8} {'stored':>8} {'synced':>8} {'exit':>8}")
            for li, l in enumerate(spec.layers):
                if int(l.op) != 3 or not tr[li, 5]:
                    continue
                e = tr[li]
                out.append(f"{li:>5} {l.name[:22]:<22} {us(e[0]):>8.1f} {us(e[1]):>8.1f} {us(e[5]):>8.1f} "
                           f"{us(e[6]):>8.1f} {us(e[11]):>8.1f} {us(e[7]):>8.1f} {us(e[8]):>8.1f} {us(e[9]):>8.1f} {us(e[10]):>8.1f} {us(e[2]):>8.1f}")
        # critical-path share per op kind in the resident run: exit(L) - exit(previous layer with a kernel)
        ex = [(li, int(tr[li, 2])) for li in range(len(spec.layers)) if tr[li, 2]]
        start = min(int(v) for v in tr[:, 0] if v)
        per = {}
        prev = start
        for li, t in ex:
            k = OPS.get(int(spec.layers[li].op), "?")
            per[k] = per.get(k, 0) + (t - prev)
            prev = t
        tot = sum(per.values())
        out.append("resident critical-path time by op (exit-to-exit increments): " +
                   ", ".join(f"{k} {v / 1e3:.1f} us ({100 * v / tot:.0f}%)" for k, v in sorted(per.items(), key=lambda kv: -kv[1])))
    text = "\n".join(out)
    print(text)
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        open(args.out, "w").write(text + "\n")


if __name__ == "__main__":
    main()
