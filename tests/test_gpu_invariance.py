"""GPU: outputs are bit-identical whatever the swap does (SURVEY §8c reading #13): claim order,
piece size, swap CTA count, cold vs resident, pipelined vs non-pipelined, SM copy vs DMA."""
import numpy as np
import pytest

from paper_2306_03622_b200 import DMA_BASELINE, ENGINE_DMA, ENGINE_SM, NO_OVERLAP, ORDER_RANDOM, ORDER_REVERSE

pytestmark = pytest.mark.gpu

SM = dict(engine=ENGINE_SM)
DMA = dict(engine=ENGINE_DMA)
CASES = [dict(), dict(order=ORDER_REVERSE, **SM), dict(order=ORDER_RANDOM, order_seed=7, **SM),
         dict(chunk_bytes=256 << 10, **SM), dict(chunk_bytes=2 << 20, **SM), dict(chunk_bytes=8 << 20, **SM),
         dict(copy_ctas=4, **SM), dict(copy_ctas=16, **SM), dict(copy_ctas=64, **SM),
         dict(flags=NO_OVERLAP), dict(flags=NO_OVERLAP, **SM), dict(flags=DMA_BASELINE),
         dict(dma_group_bytes=256 << 10, dma_streams=1, **DMA), dict(dma_group_bytes=2 << 20, dma_streams=3, **DMA),
         dict(dma_group_bytes=8 << 20, dma_streams=2, **DMA), dict(dma_group_bytes=64 << 20, dma_streams=4, **DMA)]


@pytest.mark.parametrize("name", ["bert-base", "resnet50", "gpt2-tiny", "mlp"])
def test_output_bit_identical_across_swap_modes(rt, registered, name):
    spec, w, x, mid = registered(name)
    rt.evict(mid)
    base = rt.invoke(mid, x, gpu=0).output.copy()
    warm = rt.invoke(mid, x, gpu=0)
    assert warm.stats["swap_kind"] == 0
    np.testing.assert_array_equal(warm.output, base)
    for kw in CASES:
        rt.evict(mid)
        r = rt.invoke(mid, x, gpu=0, **kw)
        np.testing.assert_array_equal(r.output, base, err_msg=str(kw))
