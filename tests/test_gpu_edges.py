"""GPU edge cases of the layer kernels against the CPU oracle: ragged GEMM shapes (M, N, K not
multiples of the 128 / 16 / 64 tiles, M just above the GEMV threshold, split-K candidates), fused
epilogues (bias, f32 / bf16 residual, every activation), the GEMV row window, convolutions on odd
image sizes through every conv path (direct 1x1, implicit GEMM with strides, im2col), attention
at T = 1 / ragged / maximum length and every head width, LayerNorm widths, and the degenerate
"no weights" table.  Integer data makes GEMMs bit-exact; random data is held to 1e-2·max|ref|."""
import numpy as np
import pytest

import oracle
from paper_2306_03622_b200 import FswError
from paper_2306_03622_b200 import fsw as F
from synth.models import DT_BF16, DT_F32, DT_I32, Act, ModelSpec, Op, Rule, f32_bits, to_bf16_bits

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel_err(got, ref):
    got = np.asarray(got, np.float64).reshape(-1)
    ref = np.asarray(ref, np.float64).reshape(-1)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30))


def run(rt, m, w=None, x=None):
    w = m.build_weights() if w is None else w
    x = m.make_input() if x is None else x
    mid = rt.register_spec(m, w)
    try:
        r = rt.invoke(mid, x, gpu=0)
        ref = oracle.output(m, w, x)
        return r.output, ref
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("M,K,N", [(9, 64, 16), (130, 72, 50), (257, 136, 33), (128, 8, 8), (200, 1000, 24),
                                   (1000, 64, 1000), (49, 4608, 40), (300, 3072, 768)])
@pytest.mark.parametrize("act,res", [(Act.NONE, None), (Act.GELU_ERF, DT_F32), (Act.RELU, DT_BF16), (Act.TANH, None),
                                     (Act.GELU_TANH, DT_F32)])
def test_gemm_ragged_shapes_and_epilogues(rt, M, K, N, act, res):
    m = ModelSpec(f"g{M}x{K}x{N}", 41, input_kind=("uniform_bf16", 1.0))
    x = m.slot("x", (M, K), DT_BF16)
    r_in = -1
    if res is not None:  # the residual comes from a second linear over the same input
        wr = m.tensor("wr", (N, K), init=("uniform", 0.05))
        r_in = m.slot("r", (M, N), res)
        m.layer(Op.LINEAR, [wr], x, -1, r_in, [Act.NONE])
    w = m.tensor("w", (N, K), init=("uniform", 0.05))
    b = m.tensor("b", (N,), init=("uniform", 0.5))
    y = m.slot("y", (M, N), DT_F32)
    m.layer(Op.LINEAR, [w, b], x, r_in, y, [act])
    m.input_slot, m.output_slot = x, y
    got, ref = run(rt, m)
    assert np.all(np.isfinite(got))
    assert rel_err(got, ref) <= TOL


@pytest.mark.parametrize("M,K,N", [(9, 64, 16), (130, 72, 50), (257, 1000, 33), (49, 4608, 512), (1000, 64, 1000)])
def test_gemm_ragged_integer_bit_exact(rt, M, K, N):
    rng = np.random.default_rng(M * 7 + N)
    m = ModelSpec("intg", 43)
    xs = m.slot("x", (M, K), DT_BF16)
    ys = m.slot("y", (M, N), DT_F32)
    w_, b_ = m.tensor("w", (N, K)), m.tensor("b", (N,))
    m.layer(Op.LINEAR, [w_, b_], xs, -1, ys, [Act.NONE])
    m.input_slot, m.output_slot = xs, ys
    W, B, X = rng.integers(-2, 3, (N, K)), rng.integers(-2, 3, N), rng.integers(-2, 3, (M, K))
    w = m.build_weights({"w": W.astype(np.float64), "b": B.astype(np.float64)})
    mid = rt.register_spec(m, w)
    try:
        out = rt.invoke(mid, to_bf16_bits(X.astype(np.float64)).view(np.uint8), gpu=0).output
        np.testing.assert_array_equal(out.reshape(M, N), (X @ W.T + B).astype(np.float32))
    finally:
        rt.unregister(mid)


@pytest.mark.parametrize("rows,r0,K,N", [(1, 0, 8, 1), (3, 2, 16, 7), (8, 0, 1000, 33), (1, 5, 2048, 1000)])
def test_gemv_row_window(rt, rows, r0, K, N):
    m = ModelSpec("gemv", 47)
    x = m.slot("x", (r0 + rows + 1, K), DT_F32)
    w = m.tensor("w", (N, K), init=("uniform", 0.1))
    b = m.tensor("b", (N,), init=("uniform", 0.5))
    y = m.slot("y", (rows, N), DT_F32)
    m.layer(Op.LINEAR, [w, b], x, -1, y, [Act.GELU_ERF, r0, rows])
    m.input_slot, m.output_slot = x, y
    got, ref = run(rt, m)
    assert rel_err(got, ref) <= TOL


@pytest.mark.parametrize("H,cin,cout,k,stride,pad", [(7, 64, 64, 3, 1, 1), (9, 64, 128, 3, 2, 1), (15, 128, 64, 1, 2, 0),
                                                     (13, 64, 32, 1, 1, 0), (11, 16, 24, 3, 1, 1), (17, 3, 16, 7, 2, 3),
                                                     (56, 64, 64, 3, 1, 1), (5, 64, 16, 5, 1, 2)])
def test_conv_paths_on_odd_sizes(rt, H, cin, cout, k, stride, pad):
    m = ModelSpec("conv", 53, input_kind=("uniform_bf16", 1.0))
    x = m.slot("img", (H, H, cin), DT_BF16)
    Ho = (H + 2 * pad - k) // stride + 1
    w = m.tensor("w", (cout, k, k, cin), init=("uniform", (3.0 / (k * k * cin)) ** 0.5))
    b = m.tensor("b", (cout,), init=("uniform", 0.1))
    r = m.slot("r", (Ho, Ho, cout), DT_BF16)
    m.layer(Op.CONV2D, [w, b], x, -1, r, [Act.RELU, stride, pad])
    w2 = m.tensor("w2", (cout, 1, 1, cout), init=("uniform", (3.0 / cout) ** 0.5))
    b2 = m.tensor("b2", (cout,), init=("uniform", 0.1))
    y = m.slot("y", (Ho, Ho, cout), DT_BF16)
    m.layer(Op.CONV2D, [w2, b2], r, r, y, [Act.NONE, 1, 0])  # 1x1 + residual
    f = m.slot("f", (1, cout), DT_F32)
    m.layer(Op.AVGPOOL, [], y, -1, f)
    m.input_slot, m.output_slot = x, f
    got, ref = run(rt, m)
    assert rel_err(got, ref) <= TOL


# T <= 128 with dh in {16, 32, 64, 128} runs the tensor-core kernel (k_attention_mma), the rest the
# scalar kernel: both against the float64 oracle
@pytest.mark.parametrize("T,H,dh,causal", [(1, 2, 64, 0), (17, 3, 8, 1), (128, 12, 64, 0), (256, 2, 128, 1),
                                           (200, 4, 32, 0), (128, 25, 64, 1), (100, 4, 32, 1), (64, 2, 128, 0),
                                           (33, 3, 16, 1), (128, 2, 128, 1), (77, 2, 64, 0), (2, 1, 16, 1)])
def test_attention_lengths_and_head_widths(rt, T, H, dh, causal):
    D = H * dh
    m = ModelSpec("attn", 59, input_kind=("uniform_bf16", 1.0))
    x = m.slot("x", (T, D), DT_BF16)
    w = m.tensor("wqkv", (3 * D, D), init=("uniform", (3.0 / D) ** 0.5))
    qkv = m.slot("qkv", (T, 3 * D), DT_BF16)
    m.layer(Op.LINEAR, [w], x, -1, qkv, [Act.NONE])
    ctx = m.slot("ctx", (T, D), DT_BF16)
    m.layer(Op.ATTENTION, [], qkv, -1, ctx, [H, dh, causal])
    wo = m.tensor("wo", (D, D), init=("uniform", (3.0 / D) ** 0.5))
    y = m.slot("y", (T, D), DT_F32)
    m.layer(Op.LINEAR, [wo], ctx, -1, y, [Act.NONE])
    m.input_slot, m.output_slot = x, y
    got, ref = run(rt, m)
    assert rel_err(got, ref) <= TOL


@pytest.mark.parametrize("rows,C", [(1, 4), (3, 100), (130, 768), (5, 2048)])
def test_layernorm_widths(rt, rows, C):
    m = ModelSpec("ln", 61)
    x = m.slot("x", (rows, C), DT_F32)
    g = m.tensor("g", (C,), init=("range", 0.9, 1.1))
    b = m.tensor("b", (C,), init=("uniform", 0.05))
    y = m.slot("y", (rows, C), DT_F32)
    m.layer(Op.LAYERNORM, [g, b], x, -1, y, [f32_bits(1e-5)])
    m.input_slot, m.output_slot = x, y
    got, ref = run(rt, m)
    assert rel_err(got, ref) <= TOL


def test_table_without_weights_is_rejected(rt):
    m = ModelSpec("noweights", 67, input_kind=("uniform_bf16", 1.0))
    x = m.slot("img", (8, 8, 16), DT_BF16)
    f = m.slot("f", (1, 16), DT_F32)
    m.layer(Op.AVGPOOL, [], x, -1, f)
    m.input_slot, m.output_slot = x, f
    with pytest.raises(FswError) as e:
        rt.register_spec(m, m.build_weights())
    assert e.value.status == F.EINVAL
