"""CPU tests of the C-ABI library (no GPU): it loads, exports every symbol include/fsw.h declares,
validates layer tables, lays out the host store (execution order, GEMM tiles), and its pool
allocator keeps SPEC's invariants (no overlap, conservation)."""
import os
import re

import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import fsw as F
from paper_2306_03622_b200 import build as B
from synth.models import DT_BF16, DT_F32, Act, ModelSpec, Op

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fsw.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fsw_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    L = F.lib()
    for s in syms:
        assert hasattr(L, s), f"libfsw.so does not export {s}"
    assert sorted(F.EXPORTS) == syms


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(F.FswError) as e:
        F.Runtime()
    assert e.value.status == F.ECUDA


# ---------------------------------------------------------------------------------------------
# pool allocator
# ---------------------------------------------------------------------------------------------
def test_arena_best_fit_coalescing_and_errors():
    a = F.Arena(1 << 20, 4096)
    x = a.alloc(100_000)     # rounds up to 102400
    y = a.alloc(200_000)
    z = a.alloc(50_000)
    assert (x, y) == (0, 102400)
    a.free(y)                # hole of 200704 between x and z
    w = a.alloc(4096)        # best fit: smallest hole that fits -> the hole after z? (tail is larger)
    assert w == 102400       # the 200704-B hole is smaller than the tail
    a.free(w)
    a.free(x)
    a.free(z)
    assert a.stats() == {"used": 0, "largest_free": 1 << 20, "n_allocated": 0}
    with pytest.raises(F.FswError) as e:
        a.free(12345)
    assert e.value.status == F.EINVAL
    with pytest.raises(F.FswError) as e:
        a.alloc(2 << 20)
    assert e.value.status == F.ENOMEM


def test_arena_random_ops_keep_invariants():
    """10^4 random alloc/free: extents never overlap and used + free space = capacity."""
    rng = np.random.default_rng(0)
    cap, align = 64 << 20, 64 << 10
    a = F.Arena(cap, align)
    live = {}
    for _ in range(10_000):
        if live and (rng.random() < 0.45 or len(live) > 200):
            off = list(live)[rng.integers(len(live))]
            a.free(off)
            del live[off]
        else:
            n = int(rng.integers(1, 4 << 20))
            try:
                off = a.alloc(n)
            except F.FswError as e:
                assert e.status == F.ENOMEM
                continue
            live[off] = (n + align - 1) // align * align
        iv = sorted(live.items())
        for (o1, s1), (o2, _) in zip(iv, iv[1:]):
            assert o1 + s1 <= o2
        st = a.stats()
        assert st["used"] == sum(live.values()) and st["n_allocated"] == len(live)
        assert st["largest_free"] <= cap - st["used"]


# ---------------------------------------------------------------------------------------------
# registration and host store (FSW_HOST_ONLY context: no GPU touched)
# ---------------------------------------------------------------------------------------------
def tiled_offsets(rows, cols, rows_pad):
    """Byte offset of W[n][k] in the tensor-core tile order, vectorised."""
    n = np.arange(rows)[:, None]
    k = np.arange(cols)[None, :]
    return ((k // 64) * (rows_pad // 8) + n // 8) * 1024 + (n % 8) * 128 + (((k % 64) // 8) ^ (n % 8)) * 16 + (k % 8) * 2


def check_store_layout(rt, mid, spec, w):
    store = rt.read_store(mid)
    info = rt.model_info(mid)
    assert store.nbytes == info["store_bytes"]
    covered = np.zeros(store.nbytes, dtype=bool)
    prev_owner = -1
    for ti, t in enumerate(spec.tensors):
        st = rt.store_tensor(mid, ti)
        src = w[t.offset:t.offset + t.nbytes]
        region = store[st["offset"]:st["offset"] + st["bytes"]]
        assert not covered[st["offset"]:st["offset"] + st["bytes"]].any(), "tensors overlap in the store"
        covered[st["offset"]:st["offset"] + st["bytes"]] = True
        assert st["offset"] % 256 == 0
        assert st["owner_layer"] >= prev_owner, "store is not in execution order"
        prev_owner = st["owner_layer"]
        if st["layout"] == 0:
            np.testing.assert_array_equal(region, src)
        else:
            rows, cols, rp, cp = st["rows"], st["cols"], st["rows_pad"], st["cols_pad"]
            assert rp % 16 == 0 and cp % 64 == 0 and st["bytes"] == rp * cp * 2
            offs = tiled_offsets(rows, cols, rp)
            vals = region.view(np.uint16)[(offs // 2).reshape(-1)]
            np.testing.assert_array_equal(vals, src.view(np.uint16))
            mask = np.ones(rp * cp, dtype=bool)
            mask[(offs // 2).reshape(-1)] = False
            assert not region.view(np.uint16)[mask].any(), "tile padding must be zero"
    assert not store[~covered].any(), "alignment padding must be zero"


@pytest.mark.parametrize("name", ["mlp-small", "bert-tiny", "gpt2-tiny", "resnet-tiny"])
def test_host_store_layout_roundtrip(name):
    spec = synth.build_model(name)
    w = spec.build_weights()
    with F.Runtime(flags=F.HOST_ONLY) as rt:
        assert rt.n_gpus == 0
        mid = rt.register_spec(spec, w)
        check_store_layout(rt, mid, spec, w)
        with pytest.raises(F.FswError) as e:
            rt.invoke(mid, spec.make_input())
        assert e.value.status == F.ECUDA


def test_full_size_store_bytes():
    """Store bytes = algorithmic bytes + alignment/tile padding (SURVEY §8a a1 byte counts)."""
    expect = {"mlp": 8_396_800, "bert-base": 218_967_556, "resnet50": 51_060_944}
    with F.Runtime(flags=F.HOST_ONLY) as rt:
        for name, alg in expect.items():
            spec = synth.build_model(name)
            assert spec.algorithmic_bytes == alg
            mid = rt.register_spec(spec, spec.build_weights())
            info = rt.model_info(mid)
            assert info["algorithmic_bytes"] == alg
            assert alg <= info["store_bytes"] <= alg * 1.002 + 64 * 1024
            rt.unregister(mid)


def _bad(mutate):
    spec = synth.build_model("bert-tiny")
    w = spec.build_weights()
    mutate(spec)
    with F.Runtime(flags=F.HOST_ONLY) as rt:
        with pytest.raises(F.FswError) as e:
            rt.register_spec(spec, w)
        return e.value.status


def test_register_rejects_bad_tables():
    def inplace(s):
        s.layers[1].out = s.layers[1].in0
    assert _bad(inplace) == F.EINVAL

    def wrong_k(s):
        s.tensors[s.layers[2].refs[0]].shape = (384, 64)
    assert _bad(wrong_k) == F.EINVAL

    def bad_slot(s):
        s.layers[3].in0 = 99
    assert _bad(bad_slot) == F.EINVAL

    def attn_dtype(s):
        s.slots[s.layers[3].in0].dtype = DT_F32
    assert _bad(attn_dtype) == F.EINVAL


def test_register_rejects_overlapping_tensors():
    spec = synth.build_model("mlp-small")
    w = spec.build_weights()
    with F.Runtime(flags=F.HOST_ONLY) as rt:
        tensors = [(t.offset, t.nbytes, t.dtype, t.shape) for t in spec.tensors]
        tensors[1] = (tensors[0][0] + 256, tensors[1][1], tensors[1][2], tensors[1][3])
        slots = [(s.dtype, s.shape) for s in spec.slots]
        refs, layers = [], []
        for l in spec.layers:
            layers.append((int(l.op), len(refs), len(l.refs), l.in0, l.in1, l.out, list(l.attr)))
            refs += list(l.refs)
        with pytest.raises(F.FswError) as e:
            rt.register("bad", w, tensors, refs, slots, layers, spec.input_slot, spec.output_slot)
        assert e.value.status == F.EINVAL


def test_unknown_model_is_enotfound():
    with F.Runtime(flags=F.HOST_ONLY) as rt:
        with pytest.raises(F.FswError) as e:
            rt.model_info(7)
        assert e.value.status == F.ENOTFOUND
        with pytest.raises(F.FswError) as e:
            rt.evict(7)
        assert e.value.status == F.ENOTFOUND


def test_tied_weight_is_stored_once():
    spec = synth.build_model("gpt2-tiny")
    w = spec.build_weights()
    with F.Runtime(flags=F.HOST_ONLY) as rt:
        mid = rt.register_spec(spec, w)
        info = rt.model_info(mid)
        wte = rt.store_tensor(mid, spec.tensor_index("wte"))
        assert wte["owner_layer"] == 0 and wte["layout"] == 0
        assert info["store_bytes"] < spec.algorithmic_bytes + 64 * 1024


# ---------------------------------------------------------------------------------------------
# generator determinism (the shared seeded-input module)
# ---------------------------------------------------------------------------------------------
def test_synth_is_deterministic_and_seeded():
    a = synth.build_model("bert-tiny").build_weights()
    b = synth.build_model("bert-tiny").build_weights()
    assert np.array_equal(a, b)
    s = synth.build_model("bert-tiny")
    s.seed = 99
    assert not np.array_equal(a, s.build_weights())
    ids = synth.build_model("bert-base").make_input().view(np.int32)
    assert ids.min() >= 0 and ids.max() < 30522 and len(np.unique(ids)) > 100


@pytest.mark.parametrize("dist,kurt", [("uniform", -1.2), ("gaussian", 0.0), ("laplace", 3.0)])
def test_synth_weight_distributions_have_the_stated_sigma_and_shape(dist, kurt):
    """bench.py's link-code runs on bell-shaped / heavy-tailed weights: same σ (0.02 for BERT's linears),
    excess kurtosis of U / N / Laplace (−1.2, 0, 3)."""
    from scipy import stats
    from synth.models import bf16_bits_to_f64
    s = synth.build_model("bert-tiny")
    s.dist = dist
    w = s.build_weights()
    t = s.tensors[s.tensor_index("embeddings.word")]
    v = bf16_bits_to_f64(w[t.offset:t.offset + t.nbytes].view(np.uint16))
    assert v.std() == pytest.approx(0.02, rel=0.02)
    assert stats.kurtosis(v) == pytest.approx(kurt, abs=0.15)


# ---------------------------------------------------------------------------------------------
# DMA engine copy plan (host logic of the swap engine)
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["bert-base", "resnet50", "mlp", "bert-tiny"])
@pytest.mark.parametrize("grp,streams", [(8 << 20, 2), (2 << 20, 1), (1 << 20, 3), (16 << 20, 4), (256, 2)])
def test_dma_plan_tiles_store_and_covers_each_layer(name, grp, streams):
    spec = synth.build_model(name)
    with F.Runtime(flags=F.HOST_ONLY) as rt:
        mid = rt.register_spec(spec, spec.build_weights())
        info = rt.model_info(mid)
        lohi, st, tg = rt.dma_plan(mid, grp, streams)
        # groups tile [0, store_bytes) contiguously in execution order, 256-B aligned
        assert lohi[0, 0] == 0 and lohi[-1, 1] == info["store_bytes"]
        assert np.all(lohi[1:, 0] == lohi[:-1, 1]) and np.all(lohi[:, 1] > lohi[:, 0])
        assert np.all(lohi % 256 == 0)
        assert np.array_equal(st, np.arange(len(st)) % streams)
        # no group exceeds a layer-merge bound: merged layers stop once >= grp, a split piece <= grp+255
        regions = []
        off = 0
        for li in range(info["n_layers"]):
            refs = [r for r in spec.layers[li].refs]
            placed = [rt.store_tensor(mid, r) for r in refs]
            mine = [p for p in placed if p["owner_layer"] == li]
            hi = max((p["offset"] + p["bytes"] for p in mine), default=None)
            regions.append(hi)
        counts = np.zeros(streams, np.int64)
        done = []   # done[g] = per-stream counts after group g landed
        for g in range(len(st)):
            counts[st[g]] += 1
            done.append(counts.copy())
        for li, hi in enumerate(regions):
            if hi is None:
                assert not tg[li].any()
                continue
            # the minimal group prefix holding the layer's last byte, expressed per stream
            g = int(np.searchsorted(lohi[:, 1], hi, side="left"))
            assert lohi[g, 0] < hi <= lohi[g, 1]
            np.testing.assert_array_equal(tg[li, :streams], done[g])
            assert not tg[li, streams:].any()
