"""GPU: the swap engine moves the host store into HBM bit-exactly (SURVEY §8c 'Swap (K1/K2)' pin),
for every model class, piece size, CTA count and claim order, and the pipeline never deadlocks."""
import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import DMA_BASELINE, ENGINE_DMA, ENGINE_SM, NO_OVERLAP, ORDER_RANDOM, ORDER_REVERSE
from synth.models import DT_BF16, DT_F32, Act, ModelSpec, Op

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine", [ENGINE_SM, ENGINE_DMA])
@pytest.mark.parametrize("name", ["mlp", "bert-base", "resnet50", "gpt2-2L"])
def test_swapped_bytes_bit_exact(rt, registered, name, engine):
    spec, w, x, mid = registered(name)
    rt.evict(mid)
    r = rt.invoke(mid, x, gpu=0, engine=engine)
    assert r.stats["swap_kind"] == 1 and r.stats["bytes_swapped"] == rt.model_info(mid)["store_bytes"]
    assert r.stats["engine"] == engine and r.stats["n_copies"] >= 1
    np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))


def _odd_model(sizes):
    """One LINEAR per size, all reading the input; weight tensors of rows x 8 bf16 (16·rows bytes)
    exercise piece / group tails that are not multiples of the piece or group size."""
    m = ModelSpec("odd", 31)
    x = m.slot("x", (1, 8), DT_F32)
    m.input_slot = x
    for i, rows in enumerate(sizes):
        wt = m.tensor(f"w{i}", (rows, 8), init=("uniform", 0.1))
        out = m.slot(f"y{i}", (1, rows), DT_F32)
        m.layer(Op.LINEAR, [wt], x, -1, out, [Act.NONE])
    m.output_slot = out
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
            rt.invoke(mid, spec.make_input(), gpu=0, chunk_bytes=chunk, copy_ctas=ctas, order=order, order_seed=chunk,
                      engine=ENGINE_SM)
            np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("grp,streams", [(256, 1), (4096, 2), (64 << 10, 4), (2 << 20, 3), (64 << 20, 2)])
def test_dma_group_and_stream_sweep_bit_exact(rt, grp, streams):
    spec = _odd_model([1, 256, 65537, 600_000])
    mid = rt.register_spec(spec, spec.build_weights())
    try:
        for flags in (0, NO_OVERLAP):
            rt.evict(mid)
            r = rt.invoke(mid, spec.make_input(), gpu=0, engine=ENGINE_DMA, dma_group_bytes=grp, dma_streams=streams,
                          flags=flags)
            assert r.stats["engine"] == ENGINE_DMA
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


@pytest.mark.parametrize("engine", [ENGINE_SM, ENGINE_DMA])
def test_swap_reaches_link_bandwidth(rt, registered, engine):
    """Sanity floor, not the bench: either swap engine sustains > 40 GB/s on BERT-base."""
    spec, w, x, mid = registered("bert-base")
    gbs = []
    for _ in range(5):
        rt.evict(mid)
        gbs.append(rt.invoke(mid, x, gpu=0, engine=engine).stats["link_gbps"])
    assert np.median(gbs) > 40.0, gbs
