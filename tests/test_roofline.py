"""CPU pins of bench.py's roofline calculator (SURVEY §8(c) 'Roofline calculator' row): the north_star
roofline against SURVEY §8(d)'s table, the flow-shop bound against SPEC.md's pipeline_latency vectors
(SPEC [OP] pipeline_latency, §4.3) and its stated bounds, and against an event simulation of
the two-stage pipeline on random instances."""
import numpy as np
import pytest

import bench
import synth


def test_pipeline_latency_spec_vectors():
    assert bench.pipeline_latency(7.0, 5.0, 1) == pytest.approx(12.0)       # N = 1: not pipelined
    assert bench.pipeline_latency(20.0, 10.0, 10) == pytest.approx(21.0)    # t_x=2, t_c=1, N=10 -> 21
    # ResNet-152 calibration: transfer 45-19 = 26 ms, compute 19 ms, 13 groups -> 27.5 ms (paper: 29)
    v = bench.pipeline_latency(26.0, 19.0, 13)
    assert v == pytest.approx(27.46, abs=0.01) and abs(v - 29.0) / 29.0 <= 0.15


def test_flowshop_equal_groups_is_spec_pipeline_latency():
    rng = np.random.default_rng(3)
    for _ in range(200):
        tx, tc, n = rng.uniform(0.1, 50), rng.uniform(0.1, 50), int(rng.integers(1, 40))
        assert bench.flowshop_ms([tx / n] * n, [tc / n] * n) == pytest.approx(bench.pipeline_latency(tx, tc, n), rel=1e-12)


def test_flowshop_bounds_and_event_simulation():
    rng = np.random.default_rng(5)
    for _ in range(500):
        n = int(rng.integers(1, 30))
        x, c = rng.exponential(1.0, n), rng.exponential(0.5, n) * (rng.uniform() < 0.8)
        t = bench.flowshop_ms(x, c)
        # SPEC "Pipeline bounds": max(transfer, compute) <= pipelined <= transfer + compute
        assert max(x.sum(), c.sum()) - 1e-12 <= t <= x.sum() + c.sum() + 1e-12
        # event simulation: layer k's compute starts when its bytes landed and layer k-1's compute ended
        land, end = 0.0, 0.0
        for k in range(n):
            land += x[k]
            end = max(end, land) + c[k]
        assert t == pytest.approx(end, rel=1e-12, abs=1e-15)


# bytes, fill and roofline T at 64 GB/s and 2.25 PF (Appendix A derivations)
SURVEY_ROWS = [  # model, store bytes, first-layer fill bytes, roofline ms, n links
    ("mlp", 8_396_800, 2_099_200, 0.164, 1),
    # SURVEY's BERT count (109,482,240 params incl. pooler) omits the QA head's 2x768 + 2 params (3,076 B)
    # that SURVEY §8(c) reading #3 adds; its "embeddings" fill (47,674,368 B) includes the embedding
    # LayerNorm, which is the second layer of the table here (first layer: the three gathered tables)
    ("bert-base", 218_964_480 + 3_076, 47_674_368 - 3_072, 4.166, 1),
    ("resnet50", 51_060_944, 18_944, 0.798, 1),
    ("gpt2-xl", 3_115_222_400, 164_099_200, 51.24, 1),
    ("gpt2-xl", 3_115_222_400, 164_099_200, 25.62, 2),
    ("gpt2-xl", 3_115_222_400, 164_099_200, 12.81, 4),
    ("gpt2-xl", 3_115_222_400, 164_099_200, 6.405, 8),
]


@pytest.mark.parametrize("name,nbytes,fill,t_roof,n", SURVEY_ROWS)
def test_roofline_matches_survey_table(name, nbytes, fill, t_roof, n):
    spec = synth.build_model(name)
    assert spec.algorithmic_bytes == nbytes
    lb = bench.layer_bytes(spec)
    assert sum(lb) == nbytes and lb[0] == fill
    t = bench.roofline_ms(nbytes, bench.model_flops(spec), lb[0], 64.0 * n, 2250.0)
    assert t == pytest.approx(t_roof, abs=5e-4 * max(1.0, t_roof))


@pytest.mark.parametrize("name,gflops", [("mlp", 8.39e-3), ("bert-base", 22.35), ("resnet50", 8.18), ("gpt2-xl", 382.7)])
def test_model_flops_match_survey_appendix(name, gflops):
    assert bench.model_flops(synth.build_model(name)) / 1e9 == pytest.approx(gflops, rel=6e-3)


def test_flowshop_of_link_bound_model_is_bytes_over_bandwidth_plus_last_compute():
    spec = synth.build_model("bert-base")
    lb = np.array(bench.layer_bytes(spec), dtype=np.float64)
    c = np.array([bench.layer_flops(spec, l) for l in spec.layers]) / (2250.0 * 1e9)
    x = lb / (64.0 * 1e6)
    t = bench.flowshop_ms(x, c)
    assert t == pytest.approx(3.421, abs=1e-3)      # SURVEY §8(d) tight flow-shop column
    assert x.sum() + c[-1] - 1e-12 <= t <= x.sum() + c.sum()
