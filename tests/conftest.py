import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# Every libfsw context the test session creates runs in poison mode (FSW_DEBUG_POISON, include/fsw.h):
# before each cold invoke the extents the swap must fill and the DMAZ staging buffer are overwritten
# with a per-invoke pattern, and before each invoke the activation workspace, so a store the swap (or a
# layer kernel) omits can never pass as a stale correct byte left by an earlier invoke of the same
# model in the same extent (the allocator hands the same offset back).
os.environ.setdefault("FSW_DEBUG_POISON", "1")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def rt():
    """One libfsw context for the whole GPU session (the pool is pre-allocated once, like the
    paper's GPU server)."""
    from paper_2306_03622_b200 import Runtime
    r = Runtime(gpu_ids=[0], pool_bytes=24 << 30)
    yield r
    r.close()


_REG = {}


@pytest.fixture(scope="session")
def registered(rt):
    """Register each synthetic model once per session: name -> (spec, weights, input, model id)."""
    import synth

    def get(name):
        if name not in _REG:
            spec = synth.build_model(name)
            w = spec.build_weights()
            x = spec.make_input()
            _REG[name] = (spec, w, x, rt.register_spec(spec, w))
        return _REG[name]
    return get
