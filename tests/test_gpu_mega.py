"""The opt-in persistent transformer kernel (k_mega, FSW_MEGA=1): one launch per invoke runs
every layer; parity with the oracle on BERT / GPT-2 models, bit-identical cold and warm outputs, a bit-exact
swap, and the cold path (the kernel waits on the swap's ready counters inside) for every swap engine.  The
switch is read once per process, so the checks run in a child process."""
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
    from paper_2306_03622_b200 import Runtime, ENGINE_SM, ENGINE_DMA, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT
    from test_gpu_parity import rel_err, TOL
    with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
        for name in ("bert-tiny", "gpt2-tiny", "bert-base", "gpt2-2L"):
            spec = synth.build_model(name)
            w, x = spec.build_weights(), spec.make_input()
            mid = rt.register_spec(spec, w, link_code=True)
            ref = oracle.output(spec, w, x)
            outs = []
            for eng in (ENGINE_SM, ENGINE_DMA, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT):
                rt.evict(mid)
                r = rt.invoke(mid, x, gpu=0, engine=eng)
                assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid)), (name, eng)
                outs.append(r.output.copy())
            rw = rt.invoke(mid, x, gpu=0)
            warm = rw.output
            assert rw.stats["n_kernels"] <= 4, ("the persistent kernel did not run", rw.stats["n_kernels"])
            for o in outs:
                assert np.array_equal(o, warm), name
            err = rel_err(warm, ref)
            assert err <= TOL, (name, err)
            print(name, "ok", err, flush=True)
            rt.unregister(mid)
""")


def test_mega_parity_every_engine_in_child_process():
    env = dict(os.environ, FSW_MEGA="1")
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count(" ok ") == 4, r.stdout
