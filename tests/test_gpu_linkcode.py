"""GPU: the link-coded engines (SMZ: zero-copy decode from the mapped coded store; DMAZ: copy-engine
DMA of coded groups into HBM staging + decode kernel) land the host store in the extent bit-exactly
(SURVEY §8c 'Swap (K1/K2)' pin) for every model class, claim order, CTA count, group size and mode,
and the outputs are bit-identical to the plain engines' (the decoded bytes are the same bytes)."""
import os
import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import (DMA_BASELINE, ENGINE_DMA, ENGINE_DMAZ, ENGINE_DMAZT, ENGINE_SM, ENGINE_SMZ, NO_OVERLAP,
                                   ORDER_RANDOM, ORDER_REVERSE, FswError)
from paper_2306_03622_b200 import fsw as F
from crafted import random_block_mixture, tier_offsets
from test_gpu_swap import _odd_model

pytestmark = pytest.mark.gpu

_CODED = {}


@pytest.fixture(scope="module")
def coded(rt, registered):
    def get(name):
        if name not in _CODED:
            spec, w, x, mid = registered(name)
            _CODED[name] = (spec, w, x, mid, rt.register_spec(spec, w, link_code=True))
        return _CODED[name]
    return get


@pytest.mark.parametrize("engine", [ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
@pytest.mark.parametrize("name", ["mlp", "bert-base", "resnet50", "gpt2-2L"])
def test_coded_swap_bit_exact_and_output_identical(rt, coded, name, engine):
    spec, w, x, plain, mid = coded(name)
    rt.evict(plain)
    base = rt.invoke(plain, x, gpu=0, engine=ENGINE_SM).output.copy()
    info = rt.model_info(mid)
    rt.evict(mid)
    r = rt.invoke(mid, x, gpu=0, engine=engine)
    assert r.stats["swap_kind"] == 1 and r.stats["engine"] == engine, r.stats
    assert r.stats["bytes_swapped"] == info["store_bytes"] and r.stats["wire_bytes"] == info["coded_bytes"]
    np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    np.testing.assert_array_equal(r.output, base)
    r2 = rt.invoke(mid, x, gpu=0)  # warm
    assert r2.stats["swap_kind"] == 0
    np.testing.assert_array_equal(r2.output, base)


def test_auto_engine_picks_coded_engines(rt, coded):
    for name, want in (("mlp", ENGINE_SMZ), ("resnet50", ENGINE_SMZ), ("bert-base", ENGINE_DMAZT)):
        spec, w, x, plain, mid = coded(name)
        rt.evict(mid)
        assert rt.invoke(mid, x, gpu=0).stats["engine"] == want
        rt.evict(plain)
        assert rt.invoke(plain, x, gpu=0).stats["engine"] in (ENGINE_SM, ENGINE_DMA)


@pytest.mark.parametrize("ctas", [1, 4, 16, 148])
def test_smz_orders_and_ctas_bit_exact(rt, ctas):
    spec = _odd_model([1, 256, 65537, 600_000])  # layer tails of 16 B .. not multiples of 1 KiB
    mid = rt.register_spec(spec, spec.build_weights(), link_code=True)
    try:
        for order in (0, ORDER_REVERSE, ORDER_RANDOM):
            for flags in (0, NO_OVERLAP):
                rt.evict(mid)
                rt.invoke(mid, spec.make_input(), gpu=0, copy_ctas=ctas, order=order, order_seed=ctas,
                          engine=ENGINE_SMZ, flags=flags)
                np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("huff", [0, 1])
@pytest.mark.parametrize("grp", [256, 4096, 64 << 10, 2 << 20, 64 << 20])
def test_dmaz_group_sweep_bit_exact(rt, grp, huff):
    """Every copy-group size, claim order and overlap mode lands bit-exactly; huff = 1 (entropy-coded pieces) runs
    the shared-memory decoder, whose claims wait for their group only when the loop reaches their ring slot
    (pending claims at every group boundary when the groups are small)."""
    spec = _odd_model([1, 256, 65537, 600_000])
    old = os.environ.get("FSW_LINK_HUFF")
    os.environ["FSW_LINK_HUFF"] = str(huff)  # read at registration
    try:
        mid = rt.register_spec(spec, spec.build_weights(), link_code=True)
    finally:
        if old is None:
            del os.environ["FSW_LINK_HUFF"]
        else:
            os.environ["FSW_LINK_HUFF"] = old
    try:
        for order, flags in ((0, 0), (0, NO_OVERLAP), (ORDER_REVERSE, 0), (ORDER_RANDOM, 0)):
            rt.evict(mid)
            r = rt.invoke(mid, spec.make_input(), gpu=0, engine=ENGINE_DMAZ, dma_group_bytes=grp, flags=flags,
                          order=order, order_seed=grp)
            assert r.stats["engine"] == ENGINE_DMAZ and r.stats["n_copies"] >= 1
            np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("n_src", [2, 3])
def test_striped_smz_virtual_sources_bit_exact(rt, coded, n_src):
    spec, w, x, plain, mid = coded("bert-base")
    rt.evict(plain)
    base = rt.invoke(plain, x, gpu=0, engine=ENGINE_SM).output.copy()
    for flags in (0, NO_OVERLAP):
        rt.evict(mid)
        r = rt.invoke(mid, x, gpu=0, stripe=[0] * n_src, flags=flags, engine=ENGINE_SMZ)
        assert r.stats["swap_kind"] == 3 and r.stats["engine"] == ENGINE_SMZ, r.stats
        # the sources read every piece's coded bytes, not the store's 128-B alignment gaps
        pcs = rt.coded_pieces(mid)
        assert r.stats["wire_bytes"] == int(pcs["cbytes"].sum()) <= rt.model_info(mid)["coded_bytes"]
        np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
        np.testing.assert_array_equal(r.output, base)


@pytest.mark.parametrize("n_src", [1, 2, 3, 4])
def test_striped_dmaz_virtual_sources_bit_exact(rt, coded, n_src):
    """DMAZ striped sources: each source copies its 4-MiB runs of the coded store with its
    copy engine into its own staging buffer and decodes them into the target (system-scope releases)."""
    spec, w, x, plain, mid = coded("bert-base")
    rt.evict(plain)
    base = rt.invoke(plain, x, gpu=0, engine=ENGINE_SM).output.copy()
    for flags in (0, NO_OVERLAP):
        rt.evict(mid)
        r = rt.invoke(mid, x, gpu=0, stripe=[0] * n_src, flags=flags, engine=ENGINE_DMAZ)
        if n_src > 1:
            assert r.stats["swap_kind"] == 3 and r.stats["engine"] == ENGINE_DMAZ, r.stats
            assert r.stats["wire_bytes"] == int(rt.coded_pieces(mid)["cbytes"].sum())
        np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
        np.testing.assert_array_equal(r.output, base)


def test_striped_dmaz_two_pool_gpus_and_dropped_run(rt):
    """Two pool GPUs on one device: pool GPU 1 is a DMAZ source of pool GPU 0.  A skipped copy run (fault
    injection, still published) must show up as wrong bytes under poison mode (negative control)."""
    from paper_2306_03622_b200 import FAULT_DROP_GROUP, FAULT_NONE, Runtime
    spec = synth.build_model("bert-base")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0, 0], pool_bytes=2 << 30) as rt2:
        mid = rt2.register_spec(spec, w, link_code=True)
        base = rt2.invoke(mid, x, gpu=0, engine=ENGINE_SM).output.copy()
        for src in ([0, 1], [1, 0], [1]):
            rt2.evict(mid)
            r = rt2.invoke(mid, x, gpu=0, stripe=src, engine=ENGINE_DMAZ)
            assert r.stats["swap_kind"] == 3
            np.testing.assert_array_equal(rt2.read_resident(mid, 0), rt2.read_store(mid))
            np.testing.assert_array_equal(r.output, base)
        rt2.evict(mid)
        rt2.set_fault(FAULT_DROP_GROUP, 3)
        try:
            rt2.invoke(mid, x, gpu=0, stripe=[0, 1], engine=ENGINE_DMAZ)
            assert not np.array_equal(rt2.read_resident(mid, 0), rt2.read_store(mid))
        finally:
            rt2.set_fault(FAULT_NONE)


@pytest.mark.parametrize("engine", [ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
def test_coded_with_cached_prefix(rt, coded, engine):
    """Partial caching (NEXT #4) + link coding: only the coded suffix moves."""
    spec, w, x, plain, mid = coded("bert-base")
    rt.evict(mid)
    base = rt.invoke(mid, x, gpu=0, engine=engine).output.copy()
    rt.evict(mid)
    kept = rt.set_cache_prefix(mid, 40 << 20)
    try:
        rt.invoke(mid, x, gpu=0, engine=engine)           # lands prefix + suffix
        rt.evict(mid, keep_prefix=True)
        r = rt.invoke(mid, x, gpu=0, engine=engine)        # moves only the suffix
        assert r.stats["bytes_swapped"] == rt.model_info(mid)["store_bytes"] - kept
        assert r.stats["wire_bytes"] < r.stats["bytes_swapped"]
        np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
        np.testing.assert_array_equal(r.output, base)
    finally:
        rt.evict(mid)
        rt.set_cache_prefix(mid, 0)


def test_coded_engine_on_plain_model_is_einval(rt, registered):
    spec, w, x, mid = registered("mlp")
    rt.evict(mid)
    for engine in (ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT):
        with pytest.raises(FswError) as e:
            rt.invoke(mid, x, gpu=0, engine=engine)
        assert e.value.status == F.EINVAL


def test_dmaz_beats_the_link(rt, coded):
    """Sanity floor, not the bench: DMAZ delivers > 60 GB/s of store bytes on BERT-base (the link
    carries ~0.76 of them at <= 55 GB/s)."""
    spec, w, x, plain, mid = coded("bert-base")
    for _ in range(5):  # untimed: the first cold invokes after registration run slower (page warm-up)
        rt.evict(mid)
        rt.invoke(mid, x, gpu=0, engine=ENGINE_DMAZ)
    gbs = []
    for _ in range(5):
        rt.evict(mid)
        gbs.append(rt.invoke(mid, x, gpu=0, engine=ENGINE_DMAZ).stats["link_gbps"])
    assert np.median(gbs) > 60.0, gbs


def _crafted_weights(spec, w, seed=11):
    """Overwrite the first weight tensor with every block kind the decoders special-case: 4-bit codes,
    one exception, > 32 exceptions (words with tiny exponents), all-zero blocks, ±0 / subnormals,
    inf / NaN exponents, and whole pieces of random 16-bit words (raw, larger than an SMZ ring slot)."""
    t = spec.tensors[0]
    words = w[t.offset:t.offset + t.nbytes].view(np.uint16)
    rng = np.random.default_rng(seed)
    sm = rng.integers(0, 256, words.size).astype(np.uint16)
    base = lambda m, e: ((m & 0x80) << 8) | (np.asarray(e).astype(np.uint16) << 7) | (m & 0x7F)
    k = 0
    words[k:k + 512] = base(sm[k:k + 512], rng.integers(100, 115, 512)); k += 512
    blk = base(sm[k:k + 512], rng.integers(101, 117, 512)); blk[5] = base(sm[k + 5], 100); words[k:k + 512] = blk; k += 512
    blk = base(sm[k:k + 512], rng.integers(120, 128, 512)); blk[::7] = base(sm[k:k + 512:7], 3); words[k:k + 512] = blk; k += 512
    words[k:k + 2048] = 0; k += 2048
    words[k:k + 512] = np.where(rng.random(512) < 0.5, 0x8000, 0) | rng.integers(0, 128, 512); k += 512
    words[k:k + 512] = base(sm[k:k + 512], rng.integers(242, 256, 512)); k += 512
    for o in range(4):  # two-tier blocks, tier-1 offset o, with escapes on both sides and exceptions
        words[k:k + 512] = base(sm[k:k + 512], 120 - tier_offsets(rng, o, n_exc=5 + 15 * o)); k += 512
    k = (k + 8191) // 8192 * 8192  # next 16-KiB piece boundary of this tensor
    words[k:k + 3 * 8192] = rng.integers(0, 1 << 16, 3 * 8192)          # three all-raw pieces
    return w


@pytest.mark.parametrize("engine", [ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
def test_coded_rare_block_kinds_bit_exact(rt, engine):
    spec = synth.build_model("mlp")
    w = _crafted_weights(spec, spec.build_weights())
    mid = rt.register_spec(spec, w, link_code=True)
    try:
        pcs = rt.coded_pieces(mid)
        hdr = pcs["hdr"].reshape(-1)
        kinds = (hdr >> 8) & 0xFF
        assert (kinds == 0xFE).any() and (kinds == 0xFF).any() and ((hdr >> 16) > 32).any()
        for o in range(4):
            assert (kinds == 0x10 + o).any()
        assert ((kinds >= 0x10) & (kinds <= 0x13) & ((hdr >> 26) > 32)).any()  # > 32 exceptions, two-tier
        assert (pcs["cbytes"] > 12288).any()  # larger than an SMZ ring slot: the direct-read fallback
        for order in (0, ORDER_REVERSE):
            rt.evict(mid)
            r = rt.invoke(mid, spec.make_input(), gpu=0, engine=engine, order=order)
            assert r.stats["engine"] == engine
            np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("engine", [ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
@pytest.mark.parametrize("seed", [1, 2])
def test_coded_random_block_mixture_bit_exact(rt, engine, seed):
    """Every block of the MLP drawn from a random mixture of block kinds (tests/crafted.py): the coded
    engines land the store bit-exactly, in execution and in reverse piece order."""
    spec = synth.build_model("mlp")
    w = random_block_mixture(spec, spec.build_weights(), seed)
    mid = rt.register_spec(spec, w, link_code=True)
    try:
        for order in (0, ORDER_REVERSE):
            rt.evict(mid)
            r = rt.invoke(mid, spec.make_input(), gpu=0, engine=engine, order=order)
            assert r.stats["engine"] == engine
            np.testing.assert_array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("tail", ["0.001", "7", "1000"])
def test_dmazt_tail_fractions_in_child_process(tail):
    """DMAZT with tails from one piece to a quarter of the coded store (FSW_DMAZT_TAIL_MB, read once per
    process): bit-exact, and the output equals the plain SM engine's, in execution and reverse order."""
    import os
    import subprocess
    import sys
    import textwrap
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = textwrap.dedent(f"""
        import sys, numpy as np
        sys.path.insert(0, {root!r})
        import synth
        from paper_2306_03622_b200 import Runtime, ENGINE_SM, ENGINE_DMAZT, ORDER_REVERSE
        spec = synth.build_model("resnet50")
        w, x = spec.build_weights(), spec.make_input()
        with Runtime(gpu_ids=[0], pool_bytes=1 << 30) as rt:
            mid = rt.register_spec(spec, w, link_code=True)
            base = rt.invoke(mid, x, gpu=0, engine=ENGINE_SM).output.copy()
            for order in (0, ORDER_REVERSE):
                rt.evict(mid)
                r = rt.invoke(mid, x, gpu=0, engine=ENGINE_DMAZT, order=order)
                assert r.stats["engine"] == ENGINE_DMAZT, r.stats
                assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
                assert np.array_equal(r.output, base)
        print("ok")
    """)
    env = dict(os.environ, FSW_DMAZT_TAIL_MB=tail)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]
