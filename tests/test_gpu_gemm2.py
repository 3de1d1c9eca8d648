"""The opt-in 2-CTA swap-AB GEMM (k_gemm2, FSW_GEMM_2CTA=1): parity with the oracle on the
transformer models whose wide linears it takes, bit-identical cold and warm outputs, and a bit-exact
swap.  The switch is read once per process, so the check runs in a child process."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent("""
    import sys, numpy as np
    sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
    import oracle, synth
    from paper_2306_03622_b200 import Runtime
    from test_gpu_parity import rel_err, TOL
    with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
        for name in ("bert-tiny", "gpt2-tiny", "bert-base", "gpt2-2L"):
            spec = synth.build_model(name)
            w, x = spec.build_weights(), spec.make_input()
            mid = rt.register_spec(spec, w)
            cold = rt.invoke(mid, x, gpu=0).output
            warm = rt.invoke(mid, x, gpu=0).output
            assert np.array_equal(cold, warm), name
            assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid)), name
            err = rel_err(cold, oracle.output(spec, w, x))
            assert err <= TOL, (name, err)
            print(name, "ok", err, flush=True)
            rt.unregister(mid)
""")


def test_gemm2_parity_in_child_process():
    env = dict(os.environ, FSW_GEMM_2CTA="1")
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count(" ok ") == 4, r.stdout
