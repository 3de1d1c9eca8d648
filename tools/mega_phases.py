"""Phase breakdown of the persistent transformer kernel (FSW_MEGA_STAMPS=1): per op, medians over CTAs of
the phases after the op's dependency resolved.   FSW_MEGA_STAMPS=1 python tools/mega_phases.py [model] [n_ops]"""
import os
import sys

os.environ.setdefault("FSW_MEGA_STAMPS", "1")
os.environ.setdefault("FSW_MEGA", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert-base"
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 16
spec = synth.build_model(name)
w, x = spec.build_weights(), spec.make_input()
KIND = {1: "gemm", 2: "ln", 3: "attn", 4: "embed", 5: "gemv"}
with Runtime(gpu_ids=[0], pool_bytes=4 << 30) as rt:
    mid = rt.register_spec(spec, w)
    for _ in range(20):
        r = rt.invoke(mid, x, gpu=0)
    print(f"{name} resident {r.stats['device_ms']:.3f} ms")
    st, ops = rt.mega_stamps(mid)
    t0 = st[st > 0].min()
    prev_done = None
    print("op kind  tasks tt sp | done(prev)->dep | dep->full1 | full1->commit | commit->accready | acc->stored | stored->done | op end")
    for i in range(min(nshow, len(ops))):
        kind, nt, tt, sp = ops[i]
        s = st[i, :nt].astype(np.float64)
        med = lambda k: float(np.median(s[:, k][s[:, k] > 0])) if (s[:, k] > 0).any() else float("nan")
        end = float(s[:, 5].max())
        if kind == 1:
            ph = [med(0), med(1), med(2), med(3), med(4), med(5)]
        else:
            ph = [med(6), float("nan"), float("nan"), float("nan"), med(7), med(5)]
        rel = lambda a, b: (a - b) / 1e3
        pd = prev_done if prev_done is not None else t0
        print(f"{i:>2} {KIND.get(int(kind), '?'):<5} {nt:>4} {tt:>3} {sp:>2} | {rel(ph[0], pd):7.2f} | {rel(ph[1], ph[0]):7.2f} | "
              f"{rel(ph[2], ph[1]):7.2f} | {rel(ph[3], ph[2]):7.2f} | {rel(ph[4], ph[3] if kind == 1 else ph[0]):7.2f} | "
              f"{rel(ph[5], ph[4]):7.2f} | {rel(end, t0):8.2f} (last done - first done {rel(end, float(s[:, 5][s[:, 5] > 0].min())):.2f})")
        prev_done = end
    # spread: per GEMM op, the slowest CTAs and where their time went
    print("\nslowest tasks per GEMM op: cta, phases (us): dep-prevdone, dep->full1, full1->commit, commit->acc, acc->stored, stored->done")
    prev_done = t0
    for i in range(min(nshow, len(ops))):
        kind, nt, tt, sp = ops[i]
        s = st[i, :nt].astype(np.float64)
        if kind == 1:
            tot = s[:, 5] - s[:, 0]
            idx = np.argsort(-s[:, 5])[:4]
            rows = []
            for c in idx:
                p = s[c]
                rows.append(f"cta {c}: " + " ".join(f"{(p[k + 1] - p[k]) / 1e3 if k >= 0 else (p[0] - prev_done) / 1e3:.2f}"
                                                    for k in [-1, 0, 1, 2, 3, 4]))
            print(f"op {i} (tt {tt} splits {sp}): " + " | ".join(rows))
            if sp == 1:
                print(f"   epilogue: acc->staged {np.median(s[:, 6] - s[:, 3]) / 1e3:.2f} us, staged->out {np.median(s[:, 7] - s[:, 6]) / 1e3:.2f} us")
            if sp > 1:
                last = s[:, 7] > 0
                print(f"   split-K: stored->flag {np.median((s[:, 6] - s[:, 4])[s[:, 6] > 0]) / 1e3:.2f} us, last arrivers "
                      f"{int(last.sum())}: flag->reduced median {np.median((s[last, 7] - s[last, 6])) / 1e3:.2f} max "
                      f"{np.max(s[last, 7] - s[last, 6]) / 1e3:.2f}, reduced->done {np.median(s[last, 5] - s[last, 7]) / 1e3:.2f} us")
        prev_done = float(s[:, 5].max())
