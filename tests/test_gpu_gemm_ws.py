"""The weight-stationary swap-AB GEMM (k_gemm_ws, gemm_ws.cu): parity with the oracle on the
transformer models and on ragged linears, for the default planner (narrow linears only), for every width
(FSW_GEMM_WS=2), for forced tilings that cover every token tile and split-K factor, and the k_gemm-only path
(FSW_GEMM_WS=0) that the default no longer takes for the narrow shapes.  Cold (every engine) and warm outputs
are bit-identical (the split-K reduction runs in split order).  The switches are read once per process, so the
checks run in child processes."""
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
    from paper_2306_03622_b200 import Runtime, ENGINE_SM, ENGINE_DMAZ
    from synth.models import DT_BF16, DT_F32, Act, ModelSpec, Op
    from test_gpu_parity import rel_err, TOL

    def ragged(M, K, N, act, res):
        m = ModelSpec(f"ws{{M}}x{{K}}x{{N}}", 43, input_kind=("uniform_bf16", 1.0))
        x = m.slot("x", (M, K), DT_BF16)
        r_in = -1
        if res is not None:
            wr = m.tensor("wr", (N, K), init=("uniform", 0.05))
            r_in = m.slot("r", (M, N), res)
            m.layer(Op.LINEAR, [wr], x, -1, r_in, [Act.NONE])
        w = m.tensor("w", (N, K), init=("uniform", 0.05))
        b = m.tensor("b", (N,), init=("uniform", 0.5))
        y = m.slot("y", (M, N), DT_F32)
        m.layer(Op.LINEAR, [w, b], x, r_in, y, [act])
        m.input_slot, m.output_slot = x, y
        return m

    specs = [synth.build_model(n) for n in ("bert-tiny", "gpt2-tiny", "bert-base", "gpt2-2L")]
    specs += [ragged(128, 768, 768, Act.GELU_ERF, DT_F32), ragged(100, 3072, 768, Act.NONE, DT_BF16),
              ragged(9, 640, 4, Act.TANH, None), ragged(77, 256, 1284, Act.RELU, DT_F32),
              ragged(128, 4608, 40, Act.GELU_TANH, None)]
    with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
        for spec in specs:
            w, x = spec.build_weights(), spec.make_input()
            mid = rt.register_spec(spec, w, link_code=True)
            ref = oracle.output(spec, w, x)
            outs = []
            for eng in (ENGINE_SM, ENGINE_DMAZ):
                rt.evict(mid)
                r = rt.invoke(mid, x, gpu=0, engine=eng)
                assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid)), spec.name
                outs.append(r.output.copy())
            warm = rt.invoke(mid, x, gpu=0).output
            for o in outs:
                assert np.array_equal(o, warm), spec.name
            err = rel_err(warm, ref)
            assert np.all(np.isfinite(warm)) and err <= TOL, (spec.name, err)
            print(spec.name, "ok", err, flush=True)
            rt.unregister(mid)
""")

N_SPECS = 9


@pytest.mark.parametrize("env", [
    {},                                   # default planner: k_gemm_ws on the narrow linears
    {"FSW_GEMM_WS": "2"},                 # every width
    {"FSW_GEMM_WS": "2", "FSW_GEMM_WS_FORCE": "16:2"},
    {"FSW_GEMM_WS": "2", "FSW_GEMM_WS_FORCE": "32:1"},
    {"FSW_GEMM_WS": "2", "FSW_GEMM_WS_FORCE": "64:4"},
    {"FSW_GEMM_WS": "2", "FSW_GEMM_WS_FORCE": "128:8"},
    {"FSW_GEMM_WS": "0"},                 # k_gemm only
    # ring mode (a few k sub-tile slots streamed through) on BERT's shapes and the ragged ones
    {"FSW_GEMM_WS": "2", "FSW_GEMM_WS_FORCE": "2304:768:64:2:2,768:768:32:1:3,3072:768:64:2:4,768:3072:64:8:2,"
                                              "768:3072:32:8:3,1296:256:32:1:2,768:4608:16:8:3,48:4608:16:8:4"},
], ids=["default", "all-widths", "tt16-s2", "tt32-s1", "tt64-s4", "tt128-s8", "k_gemm-only", "ring"])
def test_gemm_ws_parity_in_child_process(env):
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count(" ok ") == N_SPECS, r.stdout
