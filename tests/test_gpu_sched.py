"""GPU: the request scheduler (fsw_sched_*) serves submitted requests through
the swap-and-execute runtime with correct outputs and bookkeeping, and the weight pool evicts by
the heaviness-aware LRU policy."""
import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import Runtime, Scheduler

pytestmark = pytest.mark.gpu


def test_scheduler_serves_requests_with_correct_outputs():
    with Runtime(gpu_ids=[0], pool_bytes=2 << 30) as rt:
        specs = {n: synth.build_model(n) for n in ("mlp", "bert-tiny", "resnet-tiny")}
        ids, ref, inp = {}, {}, {}
        for n, sp in specs.items():
            ids[n] = rt.register_spec(sp, sp.build_weights())
            inp[n] = sp.make_input()
            ref[n] = rt.invoke(ids[n], inp[n]).output.copy()
        with Scheduler(rt, period_ms=5.0) as s:
            fids = {n: s.register_function(ids[n], deadline_ms=1000.0, p=0.98) for n in specs}
            tight = s.register_function(ids["mlp"], deadline_ms=1e-6, p=0.98)  # can never be met
            tickets = []
            for i in range(40):
                n = list(specs)[i % 3]
                out = np.empty_like(ref[n])
                tickets.append((n, fids[n], s.submit(fids[n], inp[n], out), out))
            tk = [s.submit(tight, inp["mlp"], np.empty_like(ref["mlp"])) for _ in range(5)]
            for n, fid, t, out in tickets:
                st = s.wait(t)
                assert st["rc"] == 0 and st["met_deadline"] == 1 and st["gpu"] == 0
                assert st["total_ms"] >= st["queue_ms"] >= 0
                np.testing.assert_array_equal(out, ref[n])
            for t in tk:
                assert s.wait(t)["met_deadline"] == 0
            for n, fid in fids.items():
                fs = s.function_stats(fid)
                assert fs["n"] == fs["m"] and fs["n"] in (13, 14) and fs["rrc"] < 0 and fs["queued"] == 0
            ft = s.function_stats(tight)
            assert ft["n"] == 5 and ft["m"] == 0 and ft["rrc"] == pytest.approx(0.98 * 5 / 0.02)
            st = s.stats()
            assert st["completed"] == 45 and st["met_deadline"] == 40
            assert st["n_functions"] == 4 and st["active_functions"] == 4 and st["slo_compliant_functions"] == 3
            assert st["n_resident"] + st["n_host_swaps"] == 45
            assert 0 < st["alpha"] <= 1


def test_pool_evicts_light_before_sole_copy_heavy():
    spec = synth.build_model("bert-base")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0], pool_bytes=600 << 20) as rt:   # room for two BERT-base extents
        a, b, c = (rt.register_spec(spec, w) for _ in range(3))
        rt.set_heavy(a, 0)   # light
        rt.set_heavy(b, 1)   # heavy, sole copy
        rt.set_heavy(c, 1)
        rt.invoke(b, x, gpu=0)       # b is older ...
        rt.invoke(a, x, gpu=0)       # ... than a
        assert rt.invoke(c, x, gpu=0).stats["swap_kind"] == 1   # must evict one of them
        assert rt.invoke(b, x, gpu=0).stats["swap_kind"] == 0   # the heavy sole copy stayed
        assert rt.invoke(a, x, gpu=0).stats["swap_kind"] == 1   # the light one was evicted
        rt.set_heavy(a, -1)
        assert rt.is_heavy(a)        # measured: cold / resident latency >> 1.25 at batch 1 on B200


def test_heavy_light_by_slo_in_the_runtime(rt, registered):
    """a model's class follows its measured swap time against its SLO slack — light under a
    loose deadline, heavy under a tight one (and heavy by SPEC's exec-relative rule without a deadline)."""
    spec, w, x, mid = registered("bert-tiny")
    rt.set_heavy(mid, -1)
    for _ in range(3):
        rt.evict(mid)
        rt.invoke(mid, x, gpu=0)
        rt.invoke(mid, x, gpu=0)
    rt.set_heavy_policy(0.05, 0.0)
    rt.set_slo(mid, 1000.0)        # swap (~0.05 ms) << 0.05 x ~1000 ms
    assert not rt.is_heavy(mid)
    rt.set_slo(mid, 0.3)           # tightest deadline kept: slack ~0.2 ms, 5 % of it < the swap
    assert rt.is_heavy(mid)
    rt.set_heavy(mid, 0)           # an explicit class wins
    assert not rt.is_heavy(mid)
    rt.set_heavy(mid, -1)
