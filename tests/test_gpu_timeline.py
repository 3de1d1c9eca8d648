"""GPU: the device timeline of the tracing build (libfsw_trace.so, FSW_TRACE=1) as evidence of the readiness
protocol and of the overlap: for every layer with weights, its kernel passes its weight
wait only after the last of the layer's pieces was released (never before: that would be a read of weights
that have not landed), and later layers' bytes are still arriving while earlier layers compute.  The
tracing build is a separate library, so the check runs in a child process."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent("""
    import sys, numpy as np
    sys.path.insert(0, {root!r})
    import synth
    from paper_2306_03622_b200 import Runtime, ENGINE_SM, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT
    spec = synth.build_model("bert-base")
    w, x = spec.build_weights(), spec.make_input()
    with Runtime(gpu_ids=[0], pool_bytes=2 << 30) as rt:
        mid = rt.register_spec(spec, w, link_code=True)
        for eng in (ENGINE_SM, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT):
            for _ in range(3):
                rt.evict(mid)
                r = rt.invoke(mid, x, gpu=0, engine=eng)
            tr, ti = rt.trace(mid)
            has_w = [i for i, l in enumerate(spec.layers) if l.refs]
            for i in has_w:
                entry, wait, exit_, first, last = (int(v) for v in tr[i, :5])
                assert entry and exit_ and entry <= exit_, (eng, i, tr[i])
                assert first and last and first <= last, (eng, i, tr[i])
                assert wait >= last, ("weight wait passed before the last piece was released", eng, i, wait - last)
            # overlap: some layer's kernel finished before the last piece of the model was released
            last_release = max(int(tr[i, 4]) for i in has_w)
            early = sum(1 for i in has_w if int(tr[i, 2]) < last_release)
            assert early >= len(has_w) // 2, (eng, early, len(has_w))
            print("engine", eng, "ok", early, len(has_w), flush=True)
""")


def test_timeline_wait_after_release_and_overlap():
    from paper_2306_03622_b200 import build as B
    B.build(trace=True)  # incremental: the tracing build must match the sources
    env = dict(os.environ, FSW_LIB="libfsw_trace.so", FSW_TRACE="1")
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count(" ok ") == 4, r.stdout
