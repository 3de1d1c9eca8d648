"""GPU: outputs are bit-identical whatever the swap does (SURVEY §8c reading #13): claim order,
piece size, swap CTA count, cold vs resident, pipelined vs non-pipelined, SM copy vs DMA."""
import numpy as np
import pytest

from paper_2306_03622_b200 import DMA_BASELINE, NO_OVERLAP, ORDER_RANDOM, ORDER_REVERSE

pytestmark = pytest.mark.gpu

CASES = [dict(), dict(order=ORDER_REVERSE), dict(order=ORDER_RANDOM, order_seed=7),
         dict(chunk_bytes=256 << 10), dict(chunk_bytes=2 << 20), dict(chunk_bytes=8 << 20),
         dict(copy_ctas=4), dict(copy_ctas=16), dict(copy_ctas=64),
         dict(flags=NO_OVERLAP), dict(flags=DMA_BASELINE)]


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
