"""The tcgen05 / TMEM attention kernel (k_attention_tc, attn_tc.cu; opt-in FSW_ATTN_TC=1): the
attention edge cases of test_gpu_edges.py (lengths 1..128 incl. ragged, causal and not, 2-25 heads; head width 64
runs the new kernel, the other widths and T > 128 keep the mma.sync / scalar kernels) and the transformer models
against the oracle, cold (every engine) == warm bit-identical.  The switch is read once per process, so the checks
run in child processes."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_attention_edges_with_tcgen05_kernel():
    env = dict(os.environ, FSW_ATTN_TC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-k", "attention_lengths",
                        os.path.join(ROOT, "tests", "test_gpu_edges.py")], env=env, capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "12 passed" in r.stdout, r.stdout[-1000:]


CHILD = textwrap.dedent("""
    import sys, numpy as np
    sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
    import oracle, synth
    from paper_2306_03622_b200 import Runtime, ENGINE_SM, ENGINE_DMAZ
    from test_gpu_parity import rel_err, TOL
    with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
        for name in ("bert-tiny", "gpt2-tiny", "bert-base", "gpt2-2L"):
            spec = synth.build_model(name)
            w, x = spec.build_weights(), spec.make_input()
            mid = rt.register_spec(spec, w, link_code=True)
            ref = oracle.output(spec, w, x)
            outs = []
            for eng in (ENGINE_SM, ENGINE_DMAZ):
                rt.evict(mid)
                outs.append(rt.invoke(mid, x, gpu=0, engine=eng).output.copy())
            warm = rt.invoke(mid, x, gpu=0).output
            for o in outs:
                assert np.array_equal(o, warm), name
            err = rel_err(warm, ref)
            assert err <= TOL, (name, err)
            print(name, "ok", err, flush=True)
            rt.unregister(mid)
""")


def test_models_with_tcgen05_attention():
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, FSW_ATTN_TC="1"), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count(" ok ") == 4, r.stdout
