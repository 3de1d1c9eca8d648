"""GPU: the swap engine moves the host store into HBM bit-exactly (SURVEY §8c 'Swap (K1/K2)' pin),
for every model class, piece size, CTA count and claim order, and the pipeline never deadlocks."""
import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import DMA_BASELINE, NO_OVERLAP, ORDER_RANDOM, ORDER_REVERSE
from synth.models import DT_BF16, DT_F32, Act, ModelSpec, Op

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["mlp", "bert-base", "resnet50", "gpt2-2L"])
def test_swapped_bytes_bit_exact(rt, registered, name):
    spec, w, x, mid = registered(name)
    rt.evict(mid)
    r = rt.invoke(mid, x, gpu=0)
    assert r.stats["swap_kind"] == 1 and r.stats["bytes_swapped"] == rt.model_info(mid)["store_bytes"]
    np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))


def _odd_model(sizes):
    """One LINEAR per size; weights of odd byte counts (rows*K*2 with K=8) exercise piece tails."""
    m = ModelSpec("odd", 31)
    prev = m.slot("x", (1, 8), DT_F32)
    m.input_slot = prev
    for i, rows in enumerate(sizes):
        wt = m.tensor(f"w{i}", (rows, 8), init=("uniform", 0.1))
        out = m.slot(f"y{i}", (1, rows), DT_F32)
        m.layer(Op.LINEAR, [wt], prev, -1, out, [Act.NONE])
        nxt = m.slot(f"z{i}", (1, 8), DT_F32)
        back = m.tensor(f"v{i}", (8, rows), init=("uniform", 0.1))
        m.layer(Op.LINEAR, [back], out, -1, nxt, [Act.NONE])
        prev = nxt
    m.output_slot = prev
    return m


@pytest.mark.parametrize("chunk,ctas", [(256, 1), (4096, 4), (64 << 10, 16), (2 << 20, 64), (8 << 20, 148)])
def test_piece_size_and_cta_sweep_bit_exact(rt, chunk, ctas):
    # weight tensors of 16 B, 4 KiB, ~2 MiB+16 B and ~9 MiB (rows x 8 bf16)
    spec = _odd_model([1, 256, 65537, 600_000])
    w = spec.build_weights()
    mid = rt.register_spec(spec, w)
    try:
        for order in (0, ORDER_REVERSE, ORDER_RANDOM):
            rt.evict(mid)
            rt.invoke(mid, spec.make_input(), gpu=0, chunk_bytes=chunk, copy_ctas=ctas, order=order, order_seed=chunk)
            np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("flags", [NO_OVERLAP, DMA_BASELINE, DMA_BASELINE | NO_OVERLAP])
def test_baseline_modes_bit_exact(rt, registered, flags):
    spec, w, x, mid = registered("bert-base")
    rt.evict(mid)
    r = rt.invoke(mid, x, gpu=0, flags=flags)
    assert r.stats["swap_kind"] == 1
    np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))


def test_swap_reaches_link_bandwidth(rt, registered):
    """Sanity floor, not the bench: the SM swap kernel sustains > 40 GB/s on BERT-base."""
    spec, w, x, mid = registered("bert-base")
    gbs = []
    for _ in range(5):
        rt.evict(mid)
        gbs.append(rt.invoke(mid, x, gpu=0).stats["link_gbps"])
    assert np.median(gbs) > 40.0, gbs
