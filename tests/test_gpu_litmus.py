"""GPU: the readiness protocol (DESIGN.md §5 "Memory ordering") — the evidence behind the paper's
claim that pipelined swapping "does not affect the execution order, and thus can still ensure the
correctness of the model inference" while "the transmission of subsequent layers
[overlaps] with the computation of previous layers".

fsw_debug_litmus runs each swap engine as the producer, concurrently with consumer CTAs that read
every layer exactly as a layer kernel does (acquire the layer's counter -> fence.proxy.async ->
cp.async.bulk into shared memory) and compare each 16-byte word with the host store; the destination is
poisoned before every iteration, so a release that overtakes its stores shows up as a stale word.
Negative controls: with one piece's stores dropped (still released) or one copy group skipped (still
published), the same checks must fail — poison mode makes them unconfoundable."""
import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import (ENGINE_DMA, ENGINE_DMAZ, ENGINE_DMAZT, ENGINE_SM, ENGINE_SMZ, FAULT_DROP_GROUP, FAULT_DROP_PIECE,
                                   FAULT_NONE, FswError)

pytestmark = pytest.mark.gpu

ITERS = 10_000


@pytest.fixture(scope="module")
def litmus_model(rt):
    """64 layers of 256x256 (8.4 MB): many readiness events per swap, plain and link-coded."""
    spec = synth.mlp(width=256, n_layers=64, seed=41)
    w = spec.build_weights()
    mid = rt.register_spec(spec, w, link_code=True)
    yield spec, mid
    rt.set_fault(FAULT_NONE)
    rt.unregister(mid)


@pytest.mark.parametrize("ctas", [1, 16, 148])
@pytest.mark.parametrize("engine", [ENGINE_SM, ENGINE_DMA, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
def test_litmus_release_acquire_proxy(rt, litmus_model, engine, ctas):
    spec, mid = litmus_model
    store = rt.model_info(mid)["store_bytes"]
    bad, checked = rt.litmus(mid, engine, ctas, ITERS)
    assert checked == ITERS * store, (checked, ITERS * store)
    assert bad == 0, f"{bad} stale 16-byte words seen by consumers over {ITERS} iterations"


@pytest.fixture(scope="module")
def litmus_model_huff(rt):
    """The same store with entropy-coded pieces (format v5) forced on: the shared-memory decoder as producer."""
    import os
    spec = synth.mlp(width=256, n_layers=64, seed=43)
    w = spec.build_weights()
    old = os.environ.get("FSW_LINK_HUFF")
    os.environ["FSW_LINK_HUFF"] = "1"  # read at registration
    try:
        mid = rt.register_spec(spec, w, link_code=True)
    finally:
        if old is None:
            del os.environ["FSW_LINK_HUFF"]
        else:
            os.environ["FSW_LINK_HUFF"] = old
    assert rt.coded_code(mid).any()
    yield spec, mid
    rt.set_fault(FAULT_NONE)
    rt.unregister(mid)


@pytest.mark.parametrize("ctas", [1, 16, 148])
@pytest.mark.parametrize("engine", [ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
def test_litmus_entropy_coded(rt, litmus_model_huff, engine, ctas):
    spec, mid = litmus_model_huff
    store = rt.model_info(mid)["store_bytes"]
    bad, checked = rt.litmus(mid, engine, ctas, ITERS // 4)
    assert checked == ITERS // 4 * store, (checked, ITERS // 4 * store)
    assert bad == 0, f"{bad} stale 16-byte words seen by consumers"
    rt.set_fault(FAULT_DROP_PIECE, 5)
    try:
        bad, _ = rt.litmus(mid, engine, 16, 20)
    finally:
        rt.set_fault(FAULT_NONE)
    assert bad > 0, "a dropped entropy-coded piece must be seen as stale (poison) words"


@pytest.mark.parametrize("engine", [ENGINE_SM, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
def test_litmus_negative_control_drop_piece(rt, litmus_model, engine):
    spec, mid = litmus_model
    rt.set_fault(FAULT_DROP_PIECE, 3)
    try:
        bad, checked = rt.litmus(mid, engine, 16, 20)
    finally:
        rt.set_fault(FAULT_NONE)
    assert bad > 0, "a dropped piece must be seen as stale (poison) words"


@pytest.mark.parametrize("engine", [ENGINE_DMA, ENGINE_DMAZ])
def test_litmus_negative_control_drop_group(rt, litmus_model, engine):
    spec, mid = litmus_model
    rt.set_fault(FAULT_DROP_GROUP, 2)
    try:
        bad, checked = rt.litmus(mid, engine, 16, 20)
    finally:
        rt.set_fault(FAULT_NONE)
    assert bad > 0


@pytest.mark.parametrize("engine", [ENGINE_SM, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT])
def test_dropped_piece_fails_bit_exact_check(rt, litmus_model, engine):
    """The bit-exact swap check of test_gpu_swap.py must FAIL when one piece's stores are dropped:
    the differing bytes are exactly one piece, holding the poison pattern, not stale model bytes."""
    spec, mid = litmus_model
    x = spec.make_input()
    rt.evict(mid)
    rt.invoke(mid, x, gpu=0, engine=engine)  # a correct swap first: same extent, correct bytes
    ref = rt.read_store(mid)
    assert np.array_equal(rt.read_resident(mid, 0), ref)
    rt.evict(mid)
    rt.set_fault(FAULT_DROP_PIECE, 5)
    try:
        rt.invoke(mid, x, gpu=0, engine=engine)
        got = rt.read_resident(mid, 0)
    finally:
        rt.set_fault(FAULT_NONE)
    diff = np.flatnonzero(got != ref)
    assert diff.size > 0, "dropped stores went unnoticed"
    # one piece per swap kernel (DMAZT runs two: the body's decode and the tail's), each <= 16 KiB of poison
    runs = np.split(diff, np.flatnonzero(np.diff(diff) > 16384) + 1)
    assert len(runs) <= (2 if engine == ENGINE_DMAZT else 1), [(r.min(), r.max()) for r in runs]
    for r in runs:
        lo, hi = r.min(), r.max() + 1
        assert hi - lo <= 16384, (lo, hi)
        words = got[lo & ~15: (hi + 15) & ~15].view(np.uint32)
        assert len(set((words[0::4] & 0xffff0000).tolist())) == 1  # a uniform poison pattern, not model bytes
    rt.evict(mid)
    rt.invoke(mid, x, gpu=0, engine=engine)
    assert np.array_equal(rt.read_resident(mid, 0), ref)


def test_dropped_group_fails_bit_exact_check(rt, litmus_model):
    spec, mid = litmus_model
    x = spec.make_input()
    ref = rt.read_store(mid)
    rt.evict(mid)
    rt.set_fault(FAULT_DROP_GROUP, 1)
    try:
        rt.invoke(mid, x, gpu=0, engine=ENGINE_DMA, dma_group_bytes=1 << 20)
        got = rt.read_resident(mid, 0)
    finally:
        rt.set_fault(FAULT_NONE)
    assert not np.array_equal(got, ref)
    rt.evict(mid)


def test_litmus_rejects_bad_arguments(rt, litmus_model):
    spec, mid = litmus_model
    with pytest.raises(FswError):
        rt.litmus(mid, 0, 16, 1)
    with pytest.raises(FswError):
        rt.litmus(mid, ENGINE_SM, 0, 1)
