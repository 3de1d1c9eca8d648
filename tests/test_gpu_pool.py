"""GPU: weight pool semantics — eviction by invalidation, LRU victims,
capacity errors, and the C-ABI error contract (include/fsw.h)."""
import numpy as np
import pytest

import synth
from paper_2306_03622_b200 import FswError, Runtime
from paper_2306_03622_b200 import fsw as F

pytestmark = pytest.mark.gpu


def test_evict_invalidates_without_copy_and_lru():
    spec = synth.build_model("bert-base")
    w = spec.build_weights()
    x = spec.make_input()
    store = None
    with Runtime(gpu_ids=[0], pool_bytes=600 << 20) as rt:  # holds two BERT-base extents, not three
        ids = [rt.register_spec(spec, w) for _ in range(3)]
        outs = [rt.invoke(m, x, gpu=0) for m in ids[:2]]
        assert all(o.stats["swap_kind"] == 1 for o in outs)
        st = rt.pool_stats(0)
        assert st["n_resident"] == 2 and st["n_evictions"] == 0
        assert rt.invoke(ids[0], x, gpu=0).stats["swap_kind"] == 0   # touch 0: model 1 is now LRU
        r = rt.invoke(ids[2], x, gpu=0)                                 # must evict model 1
        assert r.stats["swap_kind"] == 1
        st = rt.pool_stats(0)
        assert st["n_evictions"] == 1 and st["n_resident"] == 2
        assert rt.invoke(ids[0], x, gpu=0).stats["swap_kind"] == 0
        assert rt.invoke(ids[1], x, gpu=0).stats["swap_kind"] == 1     # evicted -> cold again,
        assert rt.pool_stats(0)["n_evictions"] == 2                    # evicting LRU model 2
        np.testing.assert_array_equal(outs[0].output, outs[1].output)
        with pytest.raises(FswError) as e:
            rt.evict(ids[2], 0)                                        # not resident any more
        assert e.value.status == F.ESTATE
        rt.evict(ids[1], 0)
        with pytest.raises(FswError) as e:
            rt.evict(ids[1], 0)
        assert e.value.status == F.ESTATE


def test_pool_too_small_is_enomem():
    spec = synth.build_model("bert-base")
    with Runtime(gpu_ids=[0], pool_bytes=128 << 20) as rt:
        mid = rt.register_spec(spec, spec.build_weights())
        with pytest.raises(FswError) as e:
            rt.invoke(mid, spec.make_input(), gpu=0)
        assert e.value.status == F.ENOMEM
        assert rt.pool_stats(0)["used"] == 0


def test_invoke_argument_errors(rt, registered):
    spec, w, x, mid = registered("bert-tiny")
    with pytest.raises(FswError) as e:
        rt.invoke(mid, x[:-4], gpu=0)
    assert e.value.status == F.EINVAL
    with pytest.raises(FswError) as e:
        rt.invoke(mid, x, out=np.empty(3, np.float32), gpu=0)
    assert e.value.status == F.EINVAL
    with pytest.raises(FswError) as e:
        rt.invoke(12345, x, gpu=0)
    assert e.value.status == F.ENOTFOUND
    bad = x.view(np.int32).copy()
    bad[5] = 10 ** 6  # token id beyond the vocabulary
    with pytest.raises(FswError) as e:
        rt.invoke(mid, bad.view(np.uint8), gpu=0)
    assert e.value.status == F.EINVAL
    r = rt.invoke(mid, x, gpu=0)          # still usable afterwards
    assert np.all(np.isfinite(r.output))


def test_unregister_then_invoke(rt):
    spec = synth.build_model("mlp-small")
    mid = rt.register_spec(spec, spec.build_weights())
    rt.invoke(mid, spec.make_input(), gpu=0)
    before = rt.pool_stats(0)["used"]
    rt.unregister(mid)
    assert rt.pool_stats(0)["used"] < before
    with pytest.raises(FswError) as e:
        rt.invoke(mid, spec.make_input(), gpu=0)
    assert e.value.status == F.ENOTFOUND


def test_public_invoke_picks_resident_gpu(rt, registered):
    spec, w, x, mid = registered("bert-tiny")
    rt.invoke(mid, x, gpu=0)
    out = np.empty(rt.model_info(mid)["output_bytes"] // 4, np.float32)
    st = rt.invoke_plain(mid, x, out)
    assert st["swap_kind"] == 0 and st["gpu"] == 0


def test_host_store_numa_node_matches_gpu(rt, registered):
    """the store's pages are bound (before first touch) to the NUMA node of the GPU
    whose host link reads them; the node comes from sysfs (-1 on single-node hosts)."""
    import os
    import subprocess
    spec, w, x, mid = registered("mlp")
    bus = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip().lower()  # 00000000:1b:00.0
    path = f"/sys/bus/pci/devices/{bus[-12:]}/numa_node"
    node = int(open(path).read()) if os.path.exists(path) else -1
    assert rt.model_info(mid)["numa_node"] == (node if node >= 0 else -1), (bus, node)
