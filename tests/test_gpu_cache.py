"""GPU: partial-parameter caching: a cached prefix of whole layers survives
evictions in its own pool extent, the next cold invoke swaps only the rest, and the swapped model
is bit-identical to the host store with an unchanged output — for every swap engine."""
import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import ENGINE_DMA, ENGINE_SM, FswError, NO_OVERLAP, Runtime
from paper_2306_03622_b200 import fsw as F

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,want", [("bert-base", 48 << 20), ("resnet50", 20 << 20), ("mlp", 3 << 20)])
def test_cached_prefix_swaps_only_the_rest(name, want):
    spec = synth.build_model(name)
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0], pool_bytes=2 << 30) as rt:
        mid = rt.register_spec(spec, w)
        base = rt.invoke(mid, x, gpu=0).output.copy()
        store = rt.read_store(mid)
        with pytest.raises(FswError) as e:
            rt.set_cache_prefix(mid, want)            # resident: evict first
        assert e.value.status == F.ESTATE
        rt.evict(mid)
        split = rt.set_cache_prefix(mid, want)
        B = rt.model_info(mid)["store_bytes"]
        assert 0 < split <= want and split < B
        r = rt.invoke(mid, x, gpu=0)                  # prefix not cached yet: everything moves
        assert r.stats["bytes_swapped"] == B
        np.testing.assert_array_equal(rt.read_resident(mid, 0), store)
        assert rt.pool_stats(0)["prefix_bytes_cached"] == split
        for kw in (dict(engine=ENGINE_SM), dict(engine=ENGINE_DMA), dict(engine=ENGINE_SM, flags=NO_OVERLAP),
                   dict(stripe=[0, 0, 0])):
            rt.evict(mid, keep_prefix=True)
            r = rt.invoke(mid, x, gpu=0, **kw)
            assert r.stats["swap_kind"] in (1, 3) and r.stats["bytes_swapped"] == B - split, (kw, r.stats)
            np.testing.assert_array_equal(rt.read_resident(mid, 0), store)
            np.testing.assert_array_equal(r.output, base, err_msg=str(kw))
        rt.evict(mid)                                 # full eviction drops the prefix too
        assert rt.pool_stats(0)["prefix_bytes_cached"] == 0
        assert rt.invoke(mid, x, gpu=0).stats["bytes_swapped"] == B
        rt.evict(mid)
        assert rt.set_cache_prefix(mid, 0) == 0


def test_pool_pressure_keeps_prefixes_until_nothing_else_is_left():
    spec = synth.build_model("bert-base")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0], pool_bytes=560 << 20) as rt:   # two BERT-base extents, not three
        a, b, c = (rt.register_spec(spec, w) for _ in range(3))
        split = rt.set_cache_prefix(a, 48 << 20)
        rt.invoke(b, x, gpu=0)                    # pool: [b][a prefix][a suffix][free]
        rt.invoke(a, x, gpu=0)
        rt.invoke(b, x, gpu=0)                    # touch b: a is the LRU model now
        r = rt.invoke(c, x, gpu=0)                # evicts a's suffix only (the hole joins the free tail)
        assert r.stats["swap_kind"] == 1
        st = rt.pool_stats(0)
        assert st["prefix_bytes_cached"] == split and st["n_resident"] == 2
        r = rt.invoke(a, x, gpu=0)                # a comes back swapping only its suffix
        assert r.stats["bytes_swapped"] == rt.model_info(a)["store_bytes"] - split
        np.testing.assert_array_equal(rt.read_resident(a, 0), rt.read_store(a))
