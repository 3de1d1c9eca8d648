"""Poisson-trace driver for the request scheduler (BASELINE.json config 5, scaled to one GPU): the
paper's "demo router" role.  Functions are distinct model instances (own seed,
own host store) of a ResNet-50 / BERT-base / GPT-2-XL mix; each function's requests arrive as a
homogeneous Poisson process with a rate drawn from U[5, 30] requests/minute (SPEC
S:52-60); deadlines 80 ms (CV) / 200 ms (BERT) at p = 0.98 and 500 ms for GPT-2-XL
(the paper has no LLM).  The GPU weight pool is capped so the working set exceeds it
and eviction runs.  Reports the SLO-compliant function ratio, per-class p50/p98 latency and the
swap-kind breakdown.

    python tools/trace.py [--functions 40] [--duration-s 60] [--pool-gb 8] [--mix 20,16,4] [--seed 42]
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2306_03622_b200 import Runtime, Scheduler  # noqa: E402

DEADLINE_MS = {"resnet50": 80.0, "bert-base": 200.0, "gpt2-xl": 500.0}


def poisson_trace(rates_per_min, duration_ms, seed):
    """Per-function homogeneous Poisson arrivals (exponential gaps), merged in time order."""
    rng = np.random.default_rng(seed)
    ev = []
    for fid, r in enumerate(rates_per_min):
        t = 0.0
        lam = r / 60000.0  # per ms
        while True:
            t += rng.exponential(1.0 / lam)
            if t > duration_ms:
                break
            ev.append((t, fid))
    ev.sort()
    return ev


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--functions", type=int, default=40)
    ap.add_argument("--mix", default="20,16,4", help="ResNet-50, BERT-base, GPT-2-XL function counts")
    ap.add_argument("--duration-s", type=float, default=60.0)
    ap.add_argument("--pool-gb", type=float, default=8.0)
    ap.add_argument("--rate-lo", type=float, default=5.0)
    ap.add_argument("--rate-hi", type=float, default=30.0)
    ap.add_argument("--p", type=float, default=0.98)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--period-ms", type=float, default=2000.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "trace.json"))
    ap.add_argument("--link-code", action="store_true", help="register every model link-coded (DESIGN.md §5b)")
    ap.add_argument("--theta", type=float, default=0.05, help="heavy iff swap > theta x SLO slack (DESIGN.md §7c)")
    ap.add_argument("--queue-budget-ms", type=float, default=0.0)
    ap.add_argument("--all-heavy", action="store_true",
                    help="force every model heavy (the paper's execution-relative rule at batch 1 on B200)")
    args = ap.parse_args()
    counts = [int(c) for c in args.mix.split(",")]
    kinds = ["resnet50"] * counts[0] + ["bert-base"] * counts[1] + ["gpt2-xl"] * counts[2]
    rng = np.random.default_rng(args.seed)
    rates = rng.uniform(args.rate_lo, args.rate_hi, len(kinds))

    rt = Runtime(gpu_ids=[0], pool_bytes=int(args.pool_gb * (1 << 30)))
    t0 = time.time()
    mids, inputs, outs = [], [], []
    for i, k in enumerate(kinds):
        spec = synth.build_model(k, seed=1000 + i)
        mids.append(rt.register_spec(spec, spec.build_weights(), link_code=args.link_code))
        inputs.append(spec.make_input())
        outs.append(rt.model_info(mids[-1])["output_bytes"])
    print(f"registered {len(kinds)} functions in {time.time() - t0:.1f}s", flush=True)

    rt.set_heavy_policy(args.theta, args.queue_budget_ms)
    if args.all_heavy:
        for m in mids:
            rt.set_heavy(m, 1)
    sched = Scheduler(rt, period_ms=args.period_ms)
    fids = [sched.register_function(m, DEADLINE_MS[k], args.p) for m, k in zip(mids, kinds)]
    heavy0 = {k: sum(rt.is_heavy(m) for m, kk in zip(mids, kinds) if kk == k) for k in set(kinds)}
    trace = poisson_trace(rates, args.duration_s * 1000.0, args.seed)
    print(f"trace: {len(trace)} requests over {args.duration_s:.0f}s ({len(trace) / args.duration_s:.1f} req/s)", flush=True)

    tickets = []
    start = time.perf_counter()
    for t_ms, fid in trace:
        delay = start + t_ms / 1000.0 - time.perf_counter()
        if delay > 0:
            time.sleep(delay)
        out = np.empty(outs[fid] // 4, np.float32)
        tickets.append((fid, sched.submit(fids[fid], inputs[fid], out)))
    res = [(fid, sched.wait(t)) for fid, t in tickets]
    wall = time.perf_counter() - start
    st = sched.stats()
    per_class = {}
    for fid, r in res:
        per_class.setdefault(kinds[fid], []).append(r["total_ms"])
    summary = {
        "functions": len(kinds), "mix": dict(zip(["resnet50", "bert-base", "gpt2-xl"], counts)),
        "link_code": args.link_code, "rates_per_min": [args.rate_lo, args.rate_hi],
        "requests": len(res), "duration_s": args.duration_s, "wall_s": round(wall, 2), "pool_gb": args.pool_gb,
        "slo_compliant_function_ratio": round(st["slo_compliant_functions"] / max(1, st["active_functions"]), 4),
        "request_deadline_ratio": round(st["met_deadline"] / max(1, st["completed"]), 4),
        "alpha_final": st["alpha"],
        "swap_kinds": {"resident": st["n_resident"], "host": st["n_host_swaps"], "peer": st["n_peer_swaps"],
                       "striped": st["n_striped_swaps"]},
        "latency_ms": {k: {"p50": round(float(np.percentile(v, 50)), 3), "p98": round(float(np.percentile(v, 98)), 3),
                           "deadline": DEADLINE_MS[k], "n": len(v)} for k, v in per_class.items()},
        "pool": rt.pool_stats(0),
        # heavy / light split: models per class before the run (estimated swap time) and
        # after it (measured), and how many evictions hit heavy models
        "heavy_policy": {"theta": args.theta, "queue_budget_ms": args.queue_budget_ms, "all_heavy": args.all_heavy},
        "heavy_models_before": heavy0,
        "heavy_models_after": {k: sum(rt.is_heavy(m) for m, kk in zip(mids, kinds) if kk == k) for k in set(kinds)},
        "models_per_kind": {k: kinds.count(k) for k in set(kinds)},
    }
    summary["eviction_mix"] = {"total": summary["pool"]["n_evictions"], "heavy": summary["pool"]["n_evictions_heavy"],
                               "light": summary["pool"]["n_evictions"] - summary["pool"]["n_evictions_heavy"]}
    print(json.dumps(summary), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(summary, open(args.out, "w"), indent=1)
    sched.close()
    rt.close()


if __name__ == "__main__":
    main()
