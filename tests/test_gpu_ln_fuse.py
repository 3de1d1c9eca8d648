"""The opt-in folded LayerNorm (FSW_LN_FUSE=1; DESIGN.md §5 "k_gemm_ws"): the GEMM that produces a LayerNorm's
input writes per-token partial statistics, the GEMM that reads its output as an operand normalises on load, the
GEMM that reads it as a residual recomputes it, and the LayerNorm launch goes.  Parity with the oracle on the
post-LN BERT models (where every LayerNorm but the last folds) and a pre-LN GPT-2, bit-identical cold / warm outputs over every swap
engine (the fused consumer also waits for the LayerNorm's own weights), fewer launches.  Read once per process:
the checks run in a child process."""
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
    # (kernels per resident invoke without the fold, LayerNorms that fold): post-LN BERT, every one but the last layer's
    # second (it feeds the pooler / QA GEMVs); pre-LN GPT-2 (2 layers), every one whose input a GEMM produces and
    # whose reader is a stationary k_gemm_ws (not the first, after the embedding, nor ln_f before the LM-head GEMV)
    expect = {{"bert-tiny": (19, 2 * 2 - 1), "bert-base": (89, 2 * 12 - 1), "gpt2-tiny": (18, 3)}}
    expect = {{n: expect[n] for n in {names!r}}}
    with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
        for name, (unfused, folded) in expect.items():
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
            for o in outs:
                assert np.array_equal(o, rw.output), name
            assert rw.stats["n_kernels"] == unfused - folded, (name, rw.stats["n_kernels"])
            err = rel_err(rw.output, ref)
            assert err <= TOL, (name, err)
            print(name, "ok", err, flush=True)
            rt.unregister(mid)
""")


# BERT-base's FFN1 / FFN2 run the ring instantiation by default (choose_ws_tiling), which the fold does not take:
# its child forces the stationary tilings of every BERT-base linear
STATIONARY_BERT_BASE = "2304:768:64:2,768:768:32:4,3072:768:64:2,768:3072:64:8"


@pytest.mark.parametrize("names,force", [(("bert-tiny", "gpt2-tiny"), None), (("bert-base",), STATIONARY_BERT_BASE)])
def test_ln_fuse_parity_every_engine_in_child_process(names, force):
    env = dict(os.environ, FSW_LN_FUSE="1")
    if force:
        env["FSW_GEMM_WS_FORCE"] = force
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), names=list(names))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count(" ok ") == len(names), r.stdout
