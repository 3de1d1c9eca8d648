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
    for _ in range(3):  # untimed warm-up
        rt.evict(mid)
        rt.invoke(mid, x, gpu=0, engine=engine)
    gbs = []
    for _ in range(5):
        rt.evict(mid)
        gbs.append(rt.invoke(mid, x, gpu=0, engine=engine).stats["link_gbps"])
    assert np.median(gbs) > 40.0, gbs


# ---------------------------------------------------------------------------------------------
# striped swap.  This box has one GPU, so the sources are the target listed several
# times: every entry runs its own swap kernel on its own stream with the protocol of a remote source
# (its share of every layer's pieces, system-scope release on the target's counters, the target's
# gate counting every source).  Bytes must land bit-exactly and the output must not change.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n_src", [2, 3, 4])
@pytest.mark.parametrize("name", ["mlp", "bert-base", "resnet50"])
def test_striped_swap_virtual_sources_bit_exact(rt, registered, name, n_src):
    spec, w, x, mid = registered(name)
    rt.evict(mid)
    base = rt.invoke(mid, x, gpu=0).output.copy()
    for flags in (0, NO_OVERLAP):
        rt.evict(mid)
        r = rt.invoke(mid, x, gpu=0, stripe=[0] * n_src, flags=flags)
        assert r.stats["swap_kind"] == 3 and r.stats["n_sources"] == n_src, r.stats
        assert r.stats["engine"] == ENGINE_SM
        np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
        np.testing.assert_array_equal(r.output, base)


def test_striped_swap_more_sources_than_pieces(rt):
    spec = _odd_model([1, 256])   # two pieces in total, four sources: two run empty shares
    mid = rt.register_spec(spec, spec.build_weights())
    try:
        r = rt.invoke(mid, spec.make_input(), gpu=0, stripe=[0, 0, 0, 0])
        assert r.stats["swap_kind"] == 3
        np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    finally:
        rt.unregister(mid)


def test_striped_swap_argument_errors(rt, registered):
    from paper_2306_03622_b200 import FswError
    from paper_2306_03622_b200 import fsw as F
    spec, w, x, mid = registered("mlp")
    rt.evict(mid)
    with pytest.raises(FswError) as e:
        rt.invoke(mid, x, gpu=0, stripe=[0, 5])     # not a GPU of the pool
    assert e.value.status == F.EINVAL
    with pytest.raises(FswError) as e:
        rt.invoke(mid, x, gpu=0, stripe=[0] * 5)    # more entries than swap slots on GPU 0
    assert e.value.status == F.EBUSY
    r = rt.invoke(mid, x, gpu=0, stripe=[0])        # one entry == target: plain host swap
    assert r.stats["swap_kind"] == 1


def test_striped_swap_two_pool_gpus_on_one_device():
    """A pool of two GPU entries mapped onto the same device: pool GPU 1 acts as a remote source
    of pool GPU 0 (its own slot, stream and ticket; stores into GPU 0's extent; system-scope
    release on GPU 0's counters).  The ctx policy stripes once the store passes stripe_min_bytes."""
    from paper_2306_03622_b200 import Runtime
    spec = synth.build_model("bert-base")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0, 0], pool_bytes=2 << 30, stripe_min_bytes=1) as rt2:
        mid = rt2.register_spec(spec, w)
        base = rt2.invoke(mid, x, gpu=0, stripe=[0]).output.copy()
        for src in ([0, 1], [1, 0], [1], [1, 1, 0]):
            rt2.evict(mid)
            r = rt2.invoke(mid, x, gpu=0, stripe=src)
            assert r.stats["swap_kind"] == 3 and r.stats["gpu"] == 0
            np.testing.assert_array_equal(rt2.read_resident(mid, 0), rt2.read_store(mid))
            np.testing.assert_array_equal(r.output, base)
        rt2.evict(mid)
        out = np.empty_like(base)
        st = rt2.invoke_plain(mid, x, out)   # policy: cold, store >= stripe_min_bytes -> striped x2
        assert st["swap_kind"] == 3 and st["n_sources"] == 2
        np.testing.assert_array_equal(out, base)


def test_peer_swap_from_resident_copy_two_pool_gpus_on_one_device():
    """Alg. 1 case 2: the model is resident on pool GPU 1 only, a cold invoke on
    GPU 0 copies it from GPU 1's extent (copy engine, device to device) instead of the host store."""
    from paper_2306_03622_b200 import NO_PEER_SWAP, FswError, Runtime
    from paper_2306_03622_b200 import fsw as F
    spec = synth.build_model("resnet50")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0, 0], pool_bytes=1 << 30) as rt2:
        mid = rt2.register_spec(spec, w)
        base = rt2.invoke(mid, x, gpu=1).output.copy()
        with pytest.raises(FswError) as e:
            rt2.invoke(mid, x, gpu=0, peer_src=0)          # the target itself
        assert e.value.status == F.EINVAL
        r = rt2.invoke(mid, x, gpu=0)                        # policy: resident on GPU 1 -> peer swap
        assert r.stats["swap_kind"] == 2 and r.stats["gpu"] == 0, r.stats
        np.testing.assert_array_equal(rt2.read_resident(mid, 0), rt2.read_store(mid))
        np.testing.assert_array_equal(r.output, base)
        rt2.evict(mid, 0)
        r = rt2.invoke(mid, x, gpu=0, peer_src=1)            # explicit
        assert r.stats["swap_kind"] == 2
        np.testing.assert_array_equal(rt2.read_resident(mid, 0), rt2.read_store(mid))
        rt2.evict(mid, 0)
        r = rt2.invoke(mid, x, gpu=0, flags=NO_PEER_SWAP)    # policy off: from the host store
        assert r.stats["swap_kind"] == 1
        np.testing.assert_array_equal(r.output, base)
        rt2.evict(mid, 1)
        rt2.evict(mid, 0)
        with pytest.raises(FswError) as e:
            rt2.invoke(mid, x, gpu=0, peer_src=1)          # not resident on GPU 1 any more
        assert e.value.status == F.ESTATE


def test_striped_swap_numa_dealing_two_fake_nodes(monkeypatch):
    """FSW_FAKE_NUMA=2: pool GPU i pretends to sit on NUMA node i % 2, so the host stores are mapped
    chunk-wise across two nodes and striped swaps deal each chunk to a source on its node (no mbind on
    this single-node box).  Bytes and outputs must not change, plain and link-coded."""
    from paper_2306_03622_b200 import ENGINE_SMZ, Runtime
    monkeypatch.setenv("FSW_FAKE_NUMA", "2")
    spec = synth.build_model("bert-base")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0, 0], pool_bytes=2 << 30, stripe_min_bytes=1) as rt2:
        plain = rt2.register_spec(spec, w)
        coded = rt2.register_spec(spec, w, link_code=True)
        assert rt2.model_info(plain)["numa_node"] == -2
        base = rt2.invoke(plain, x, gpu=0, stripe=[0]).output.copy()
        for mid, eng in ((plain, 0), (coded, ENGINE_SMZ)):
            for src in ([0, 1], [1, 0], [0, 1, 1]):
                rt2.evict(mid)
                r = rt2.invoke(mid, x, gpu=0, stripe=src, engine=eng)
                assert r.stats["swap_kind"] == 3
                np.testing.assert_array_equal(rt2.read_resident(mid, 0), rt2.read_store(mid))
                np.testing.assert_array_equal(r.output, base)


def test_peer_swap_never_reads_an_extent_still_being_swapped_in():
    """while thread A cold-loads a model onto pool GPU 0, a concurrent invoke on pool
    GPU 1 must not treat GPU 0's half-written extent as a resident copy (Algorithm 1 case 2 needs a
    complete copy): it swaps from the host, and both copies end up bit-exact."""
    import threading
    import time
    from paper_2306_03622_b200 import ENGINE_SM, Runtime
    spec = synth.build_model("bert-base")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0, 0], pool_bytes=2 << 30) as rt2:
        mid = rt2.register_spec(spec, w)
        base = rt2.invoke(mid, x, gpu=0).output.copy()
        for _ in range(5):
            rt2.evict(mid)
            res = {}

            def run(gpu, delay):
                time.sleep(delay)
                res[gpu] = rt2.invoke(mid, x, gpu=gpu, engine=ENGINE_SM, chunk_bytes=16 << 10)

            ta = threading.Thread(target=run, args=(0, 0.0))
            tb = threading.Thread(target=run, args=(1, 0.001))  # A's swap takes ~4 ms
            ta.start(); tb.start(); ta.join(); tb.join()
            assert res[0].stats["swap_kind"] == 1
            assert res[1].stats["swap_kind"] in (1, 2)  # peer only if A had completed first
            for g in (0, 1):
                np.testing.assert_array_equal(rt2.read_resident(mid, g), rt2.read_store(mid))
                np.testing.assert_array_equal(res[g].output, base)
