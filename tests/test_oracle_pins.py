"""Pins for the oracle (CPU, no GPU): each check ties oracle/oracle.c to something other than
itself — textbook constants, closed forms, exact integer brute force, or an independent
library implementation (torch float64 functional ops).  DESIGN.md §"Oracle pins" lists which
pin covers which function.
"""
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth
from synth.models import (DT_BF16, DT_F32, DT_I32, Act, ModelSpec, Op, Rule, bf16_bits_to_f64,
                          f32_bits, to_bf16_bits)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def bf16_round(a):
    return bf16_bits_to_f64(to_bf16_bits(np.asarray(a, dtype=np.float64))).reshape(np.shape(a))


# ---------------------------------------------------------------------------------------------
# scalar activations
# ---------------------------------------------------------------------------------------------
def test_gelu_erf_textbook_normal_cdf():
    """GELU(x) = x·Φ(x); Φ from a printed table (tests/golden/normal_cdf.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "normal_cdf.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) >= 5
    for x, phi in rows:
        x, phi = float(x), float(phi)
        assert oracle.gelu_erf(x) == pytest.approx(x * phi, rel=1e-14, abs=1e-16)


def test_gelu_tanh_matches_torch_tanh_approximation():
    for x in [-3.0, -1.0, -0.1, 0.0, 0.3, 1.0, 2.5]:
        ref = F.gelu(torch.tensor(x, dtype=torch.float64), approximate="tanh").item()
        assert oracle.gelu_tanh(x) == pytest.approx(ref, rel=1e-14, abs=1e-16)
    assert oracle.gelu_tanh(1.0) == pytest.approx(0.8411919906082768, rel=1e-14)


# ---------------------------------------------------------------------------------------------
# single-op models
# ---------------------------------------------------------------------------------------------
def _one_layer(op, in_shape, out_shape, in_dt=DT_F32, out_dt=DT_F32):
    m = ModelSpec("one", 99)
    m.slot("in", in_shape, in_dt)
    m.slot("out", out_shape, out_dt)
    m.input_slot, m.output_slot = 0, 1
    return m


def _f32_input(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32)).view(np.uint8)


def test_layernorm_constant_row_gives_beta():
    m = _one_layer(Op.LAYERNORM, (3, 16), (3, 16))
    g = m.tensor("g", (16,), init=("range", 0.5, 1.5))
    b = m.tensor("b", (16,), init=("uniform", 0.3))
    m.layer(Op.LAYERNORM, [g, b], 0, -1, 1, [f32_bits(1e-5)])
    w = m.build_weights()
    x = np.full((3, 16), 2.75, dtype=np.float32)
    y = oracle.output(m, w, _f32_input(x))
    beta = bf16_bits_to_f64(w[m.tensors[b].offset:m.tensors[b].offset + 32].view(np.uint16))
    np.testing.assert_array_equal(y, np.broadcast_to(beta, (3, 16)))


def test_layernorm_alternating_closed_form():
    """x = ±a alternating: μ = 0, σ² = a² ⇒ y = ±γ·a/√(a²+eps) (+β = 0)."""
    m = _one_layer(Op.LAYERNORM, (1, 8), (1, 8))
    g = m.tensor("g", (8,), init=("ones",))
    b = m.tensor("b", (8,), init=("zeros",))
    eps = 1e-5
    m.layer(Op.LAYERNORM, [g, b], 0, -1, 1, [f32_bits(eps)])
    w = m.build_weights()
    x = np.array([[1, -1] * 4], dtype=np.float32)
    y = oracle.output(m, w, _f32_input(x))
    e32 = float(np.float32(eps))
    np.testing.assert_allclose(y[0], [1 / math.sqrt(1 + e32), -1 / math.sqrt(1 + e32)] * 4, rtol=1e-15)
    assert y[0, 0] == pytest.approx(0.999995000037, rel=1e-11)


def test_layernorm_vs_torch_float64():
    rng = np.random.default_rng(0)
    m = _one_layer(Op.LAYERNORM, (5, 96), (5, 96))
    g = m.tensor("g", (96,), init=("range", 0.9, 1.1))
    b = m.tensor("b", (96,), init=("uniform", 0.05))
    m.layer(Op.LAYERNORM, [g, b], 0, -1, 1, [f32_bits(1e-12)])
    w = m.build_weights()
    x = rng.standard_normal((5, 96)).astype(np.float32)
    y = oracle.output(m, w, _f32_input(x))
    gam = torch.tensor(bf16_bits_to_f64(w[m.tensors[g].offset:][:192].view(np.uint16)))
    bet = torch.tensor(bf16_bits_to_f64(w[m.tensors[b].offset:][:192].view(np.uint16)))
    ref = F.layer_norm(torch.tensor(x, dtype=torch.float64), (96,), gam, bet, eps=float(np.float32(1e-12)))
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-13, atol=1e-13)


def test_linear_identity_and_zero_closed_forms():
    n = 64
    m = _one_layer(Op.LINEAR, (1, n), (1, n))
    w_ = m.tensor("w", (n, n))
    b_ = m.tensor("b", (n,))
    m.layer(Op.LINEAR, [w_, b_], 0, -1, 1, [Act.NONE])
    x = np.linspace(-1, 1, n, dtype=np.float32).reshape(1, n)
    w = m.build_weights({"w": np.eye(n), "b": np.zeros(n)})
    np.testing.assert_array_equal(oracle.output(m, w, _f32_input(x)), x.astype(np.float64))
    bias = np.arange(n) * 0.25 - 3
    w = m.build_weights({"w": np.zeros((n, n)), "b": bias})
    np.testing.assert_array_equal(oracle.output(m, w, _f32_input(x)), bias.reshape(1, n))


def test_linear_row_selection_and_residual():
    """LINEAR with a row window (pooler / LM-head use) and a residual input, vs float64 brute force."""
    rng = np.random.default_rng(1)
    m = ModelSpec("rows", 5)
    xs = m.slot("x", (6, 32), DT_F32)
    rs = m.slot("r", (2, 16), DT_F32)
    ys = m.slot("y", (2, 16), DT_F32)
    w_ = m.tensor("w", (16, 32))
    b_ = m.tensor("b", (16,))
    m.layer(Op.LINEAR, [w_, b_], xs, rs, ys, [Act.RELU, 3, 2])
    m.input_slot, m.output_slot = xs, ys
    W = rng.integers(-3, 4, (16, 32)).astype(np.float64)
    B = rng.integers(-3, 4, 16).astype(np.float64)
    X = rng.integers(-2, 3, (6, 32)).astype(np.float32)
    R = rng.integers(-5, 6, (2, 16)).astype(np.float64)
    w = m.build_weights({"w": W, "b": B})
    y = oracle.forward(m, w, _f32_input(X), slots={rs: R})[ys]
    ref = np.maximum(X[3:5].astype(np.int64) @ W.astype(np.int64).T + B.astype(np.int64) + R.astype(np.int64), 0)
    np.testing.assert_array_equal(y, ref)


def integer_mlp_weights(spec, seed):
    """SURVEY §8c 'Integer-exact MLPs': ≤4 non-zeros per row in {−1,+1}, biases in {−1,0,1}."""
    rng = np.random.default_rng(seed)
    ov = {}
    for i, l in enumerate(spec.layers):
        wt = spec.tensors[l.refs[0]]
        n_out, n_in = wt.shape
        W = np.zeros((n_out, n_in))
        for o in range(n_out):
            cols = rng.choice(n_in, size=4, replace=False)
            W[o, cols] = rng.choice([-1.0, 1.0], size=4)
        ov[wt.name] = W
        ov[spec.tensors[l.refs[1]].name] = rng.integers(-1, 2, n_out).astype(np.float64)
    return ov


def test_integer_mlp_full_shape_exact_vs_int64_brute_force():
    """4×1024 MLP with ReLU/identity: oracle == int64 brute force bit-exactly at the real shape."""
    spec = synth.mlp(width=1024, n_layers=4, act=Act.RELU, seed=21)
    ov = integer_mlp_weights(spec, 21)
    w = spec.build_weights(ov)
    x = np.random.default_rng(3).integers(-1, 2, (1, 1024)).astype(np.float32)
    y = oracle.output(spec, w, _f32_input(x))
    h = x.astype(np.int64)
    for i, l in enumerate(spec.layers):
        W = ov[spec.tensors[l.refs[0]].name].astype(np.int64)
        b = ov[spec.tensors[l.refs[1]].name].astype(np.int64)
        h = h @ W.T + b
        if i < 3:
            h = np.maximum(h, 0)
    np.testing.assert_array_equal(y, h.astype(np.float64))


def test_mlp_identity_gelu_closed_form():
    """W = I, b = 0, GELU on the hidden layers ⇒ y = GELU(GELU(GELU(x))) elementwise (4-layer MLP)."""
    n = 32
    spec = synth.mlp(width=n, n_layers=4, act=Act.GELU_ERF)
    ov = {}
    for l in spec.layers:
        ov[spec.tensors[l.refs[0]].name] = np.eye(n)
        ov[spec.tensors[l.refs[1]].name] = np.zeros(n)
    w = spec.build_weights(ov)
    x = np.linspace(-2, 2, n, dtype=np.float32).reshape(1, n)
    y = oracle.output(spec, w, _f32_input(x))
    phi = lambda v: 0.5 * (1 + math.erf(v / math.sqrt(2)))
    for i in range(n):
        v = float(x[0, i])
        for _ in range(3):
            v = v * phi(v)
        assert y[0, i] == pytest.approx(v, rel=1e-14, abs=1e-300)


def test_random_small_mlp_vs_float64_torch():
    spec = synth.build_model("mlp-small")
    w = spec.build_weights()
    x = spec.make_input()
    y = oracle.output(spec, w, x)
    h = torch.tensor(x.view(np.float32).astype(np.float64)).reshape(1, -1)
    for i, l in enumerate(spec.layers):
        Wt, bt = spec.tensors[l.refs[0]], spec.tensors[l.refs[1]]
        W = torch.tensor(bf16_bits_to_f64(w[Wt.offset:Wt.offset + Wt.nbytes].view(np.uint16)).reshape(Wt.shape))
        b = torch.tensor(bf16_bits_to_f64(w[bt.offset:bt.offset + bt.nbytes].view(np.uint16)))
        h = F.linear(h, W, b)
        if i < len(spec.layers) - 1:
            h = F.gelu(h)
    np.testing.assert_allclose(y, h.numpy(), rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------------------------
# attention
# ---------------------------------------------------------------------------------------------
def _attn_model(T, H, dh, causal):
    m = _one_layer(Op.ATTENTION, (T, 3 * H * dh), (T, H * dh))
    m.layer(Op.ATTENTION, [], 0, -1, 1, [H, dh, int(causal)])
    return m


@pytest.mark.parametrize("causal", [False, True])
def test_attention_uniform_softmax_is_mean_or_prefix_mean(causal):
    """q = k = 0 ⇒ softmax uniform ⇒ ctx = mean of V rows (bidirectional) or prefix mean (causal)."""
    T, H, dh = 128, 2, 8
    rng = np.random.default_rng(4)
    qkv = np.zeros((T, 3 * H * dh), dtype=np.float32)
    qkv[:, 2 * H * dh:] = rng.standard_normal((T, H * dh))
    y = oracle.output(_attn_model(T, H, dh, causal), np.zeros(0, np.uint8), _f32_input(qkv))
    v = qkv[:, 2 * H * dh:].astype(np.float64)
    if causal:
        ref = np.cumsum(v, axis=0) / np.arange(1, T + 1)[:, None]
    else:
        ref = np.broadcast_to(v.mean(axis=0), (T, H * dh))
    np.testing.assert_allclose(y, ref, rtol=1e-13, atol=1e-14)


def test_attention_known_probabilities_pin_scale_and_operands():
    """One head, T=3, dh=4: choose q·k_j/√dh = [0, ln 2, ln 5] ⇒ P = [1/8, 2/8, 5/8] exactly.
    Any dropped scale, transposed q/k, or head-offset error changes the mixture of v rows."""
    T, dh = 3, 4
    qkv = np.zeros((T, 3 * dh), dtype=np.float64)
    q = np.array([2.0, 0, 0, 0])           # √dh = 2 ⇒ score_j = k_j[0]
    qkv[:, 0:dh] = q
    qkv[0, dh:2 * dh] = [0.0, 9, 9, 9]          # k rows: only k[0] matters (q has a single non-zero)
    qkv[1, dh:2 * dh] = [math.log(2), -7, 1, 2]
    qkv[2, dh:2 * dh] = [math.log(5), 3, 3, 3]
    V = np.array([[8.0, 0, 0, 1], [0, 8, 0, 1], [0, 0, 8, 1]])
    qkv[:, 2 * dh:] = V
    m = _attn_model(T, 1, dh, False)
    m.slots[0].dtype = DT_F32
    inp = np.ascontiguousarray(qkv.astype(np.float32))
    y = oracle.output(m, np.zeros(0, np.uint8), inp.view(np.uint8))
    k0 = inp[:, dh].astype(np.float64)  # float32-rounded log constants
    p = np.exp(k0) / np.exp(k0).sum()
    np.testing.assert_allclose(p, [1 / 8, 2 / 8, 5 / 8], rtol=1e-6)
    np.testing.assert_allclose(y[0], p @ V, rtol=1e-14)
    np.testing.assert_allclose(y[0], [1, 2, 5, 1], rtol=1e-6)


@pytest.mark.parametrize("causal", [False, True])
def test_attention_vs_torch_sdpa_float64(causal):
    T, H, dh = 17, 3, 16
    rng = np.random.default_rng(5)
    qkv = rng.standard_normal((T, 3 * H * dh)).astype(np.float32)
    y = oracle.output(_attn_model(T, H, dh, causal), np.zeros(0, np.uint8), _f32_input(qkv))
    t = torch.tensor(qkv, dtype=torch.float64)
    q, k, v = (t[:, i * H * dh:(i + 1) * H * dh].reshape(T, H, dh).transpose(0, 1) for i in range(3))
    ref = F.scaled_dot_product_attention(q, k, v, is_causal=causal).transpose(0, 1).reshape(T, H * dh)
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------------------------------------------
# convolution and pooling
# ---------------------------------------------------------------------------------------------
def _conv_model(Hin, cin, cout, k, stride, pad, act=Act.NONE, res=False):
    m = ModelSpec("conv", 7)
    xi = m.slot("x", (Hin, Hin, cin), DT_F32)
    Ho = (Hin + 2 * pad - k) // stride + 1
    r = m.slot("r", (Ho, Ho, cout), DT_F32) if res else -1
    yo = m.slot("y", (Ho, Ho, cout), DT_F32)
    w_ = m.tensor("w", (cout, k, k, cin), init=("uniform", 0.3))
    b_ = m.tensor("b", (cout,), init=("uniform", 0.3))
    m.layer(Op.CONV2D, [w_, b_], xi, r, yo, [act, stride, pad])
    m.input_slot, m.output_slot = xi, yo
    return m, r


def test_conv_delta_kernel_is_identity():
    m, _ = _conv_model(9, 4, 4, 3, 1, 1)
    W = np.zeros((4, 3, 3, 4))
    for c in range(4):
        W[c, 1, 1, c] = 1.0
    w = m.build_weights({"w": W, "b": np.zeros(4)})
    x = np.random.default_rng(6).standard_normal((9, 9, 4)).astype(np.float32)
    np.testing.assert_array_equal(oracle.output(m, w, _f32_input(x)), x.astype(np.float64))


def test_conv_all_ones_tap_counts():
    """All-ones 3×3 p1 on all-ones input ⇒ 4·C at corners, 6·C on edges, 9·C inside (pins padding)."""
    C = 5
    m, _ = _conv_model(6, C, 2, 3, 1, 1)
    w = m.build_weights({"w": np.ones((2, 3, 3, C)), "b": np.zeros(2)})
    y = oracle.output(m, w, _f32_input(np.ones((6, 6, C))))
    assert y[0, 0, 0] == 4 * C and y[5, 5, 1] == 4 * C
    assert y[0, 3, 0] == 6 * C and y[2, 0, 1] == 6 * C
    assert np.all(y[1:5, 1:5] == 9 * C)


def test_resnet50_output_sizes():
    m = synth.resnet50()
    shp = {s.name: s.shape for s in m.slots}
    assert shp["conv1.out"] == (112, 112, 64)
    assert shp["maxpool.out"] == (56, 56, 64)
    assert shp["layer2.0.conv3.out"] == (28, 28, 512)
    assert shp["layer3.0.conv3.out"] == (14, 14, 1024)
    assert shp["layer4.2.conv3.out"] == (7, 7, 2048)
    assert m.param_count == 25_530_472 and m.algorithmic_bytes == 51_060_944


@pytest.mark.parametrize("k,stride,pad,act,res", [(3, 1, 1, Act.RELU, True), (7, 2, 3, Act.NONE, False),
                                                   (1, 2, 0, Act.NONE, False), (1, 1, 0, Act.RELU, True)])
def test_conv_vs_torch_conv2d_float64(k, stride, pad, act, res):
    m, rslot = _conv_model(11, 6, 5, k, stride, pad, act, res)
    w = m.build_weights()
    rng = np.random.default_rng(7)
    x = rng.standard_normal((11, 11, 6)).astype(np.float32)
    Ho = m.slots[m.output_slot].shape[0]
    R = rng.standard_normal((Ho, Ho, 5)) if res else None
    y = oracle.forward(m, w, _f32_input(x), slots={rslot: R} if res else None)[m.output_slot]
    Wt, bt = m.tensors[0], m.tensors[1]
    W = torch.tensor(bf16_bits_to_f64(w[Wt.offset:Wt.offset + Wt.nbytes].view(np.uint16)).reshape(Wt.shape))
    b = torch.tensor(bf16_bits_to_f64(w[bt.offset:bt.offset + bt.nbytes].view(np.uint16)))
    xt = torch.tensor(x, dtype=torch.float64).permute(2, 0, 1)[None]
    ref = F.conv2d(xt, W.permute(0, 3, 1, 2), b, stride=stride, padding=pad)[0].permute(1, 2, 0)
    if res:
        ref = ref + torch.tensor(R)
    if act == Act.RELU:
        ref = torch.relu(ref)
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-12, atol=1e-12)


def test_maxpool_and_avgpool_vs_torch():
    m = ModelSpec("pool", 8)
    xi = m.slot("x", (13, 13, 3), DT_F32)
    mp = m.slot("mp", (7, 7, 3), DT_F32)
    ap = m.slot("ap", (1, 3), DT_F32)
    m.layer(Op.MAXPOOL, [], xi, -1, mp, [3, 2, 1])
    m.layer(Op.AVGPOOL, [], mp, -1, ap)
    m.input_slot, m.output_slot = xi, ap
    x = np.random.default_rng(8).standard_normal((13, 13, 3)).astype(np.float32)
    out = oracle.forward(m, np.zeros(0, np.uint8), _f32_input(x))
    xt = torch.tensor(x, dtype=torch.float64).permute(2, 0, 1)[None]
    ref = F.max_pool2d(xt, 3, 2, 1)[0].permute(1, 2, 0)
    np.testing.assert_array_equal(out[mp], ref.numpy())
    np.testing.assert_allclose(out[ap][0], ref.numpy().mean(axis=(0, 1)), rtol=1e-14)


# ---------------------------------------------------------------------------------------------
# embeddings
# ---------------------------------------------------------------------------------------------
def test_embed_gathers_rows():
    m = ModelSpec("emb", 9)
    ids = m.slot("ids", (4,), DT_I32)
    out = m.slot("e", (4, 8), DT_F32)
    a = m.tensor("word", (10, 8))
    b = m.tensor("pos", (6, 8))
    c = m.tensor("type", (2, 8))
    m.layer(Op.EMBED, [a, b, c], ids, -1, out, [3, Rule.IDS, Rule.POSITION, Rule.ZERO])
    m.input_slot, m.output_slot = ids, out
    word = np.arange(80).reshape(10, 8) * 0.5
    pos = -np.arange(48).reshape(6, 8)
    typ = np.arange(16).reshape(2, 8) * 100.0
    w = m.build_weights({"word": word, "pos": pos, "type": typ})
    idv = np.array([7, 0, 9, 7], dtype=np.int32)
    y = oracle.output(m, w, idv.view(np.uint8))
    ref = word[idv] + pos[:4] + typ[0]
    np.testing.assert_array_equal(y, ref)


# ---------------------------------------------------------------------------------------------
# whole networks: closed forms (SURVEY §8c "Whole-network closed forms")
# ---------------------------------------------------------------------------------------------
def _zero_linear_overrides(spec, keep_qa_bias=True):
    ov = {}
    for l in spec.layers:
        if l.op in (Op.LINEAR, Op.CONV2D):
            for r in l.refs:
                t = spec.tensors[r]
                if t.name in ("wte",):
                    continue
                if keep_qa_bias and t.name in ("qa.bias", "fc.bias"):
                    continue
                ov[t.name] = np.zeros(t.shape)
    return ov


def _t(w, spec, name):
    t = spec.tensors[spec.tensor_index(name)]
    return bf16_bits_to_f64(w[t.offset:t.offset + t.nbytes].view(np.uint16)).reshape(t.shape)


def _ln(x, g, b, eps):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def test_bert_zero_linears_closed_form():
    """All Linear W,b = 0 ⇒ attention output 0, every sublayer is x ↦ LN(x); QA logits = b_qa."""
    spec = synth.build_model("bert-tiny")
    w = spec.build_weights(_zero_linear_overrides(spec))
    ids = spec.make_input()
    out = oracle.forward(spec, w, ids)
    np.testing.assert_array_equal(out[spec.output_slot], np.broadcast_to(_t(w, spec, "qa.bias"), (64, 2)))
    e = _t(w, spec, "embeddings.word")[ids.view(np.int32)] + _t(w, spec, "embeddings.position")[:64] + \
        _t(w, spec, "embeddings.token_type")[0]
    eps = float(np.float32(1e-12))
    x = _ln(e, _t(w, spec, "embeddings.ln.gamma"), _t(w, spec, "embeddings.ln.beta"), eps)
    for i in range(2):
        x = _ln(x, _t(w, spec, f"layer{i}.ln1.gamma"), _t(w, spec, f"layer{i}.ln1.beta"), eps)
        x = _ln(x, _t(w, spec, f"layer{i}.ln2.gamma"), _t(w, spec, f"layer{i}.ln2.beta"), eps)
    np.testing.assert_allclose(out[spec.slots.index(next(s for s in spec.slots if s.name == "x"))], x,
                               rtol=1e-12, atol=1e-12)


def test_gpt_zero_linears_closed_form():
    """All Linear W,b = 0 (LM head tied to wte kept) ⇒ residual passes through ⇒
    logits = LN_f(wte[id_last] + wpe[last]) · wteᵀ."""
    spec = synth.build_model("gpt2-tiny")
    w = spec.build_weights(_zero_linear_overrides(spec))
    ids = spec.make_input().view(np.int32)
    y = oracle.output(spec, w, ids.view(np.uint8))
    wte, wpe = _t(w, spec, "wte"), _t(w, spec, "wpe")
    x = wte[ids[-1]] + wpe[len(ids) - 1]
    xf = _ln(x, _t(w, spec, "ln_f.gamma"), _t(w, spec, "ln_f.beta"), float(np.float32(1e-5)))
    np.testing.assert_allclose(y[0], wte @ xf, rtol=1e-11, atol=1e-12)


def test_resnet_zero_convs_gives_fc_bias():
    spec = synth.build_model("resnet-tiny")
    w = spec.build_weights(_zero_linear_overrides(spec))
    y = oracle.output(spec, w, spec.make_input())
    np.testing.assert_array_equal(y[0], _t(w, spec, "fc.bias"))


# ---------------------------------------------------------------------------------------------
# whole networks vs independent library implementations (float64)
# ---------------------------------------------------------------------------------------------
def test_bert_tiny_vs_hf_transformers_float64():
    from transformers import BertConfig, BertForQuestionAnswering
    spec = synth.build_model("bert-tiny")
    w = spec.build_weights()
    ids = spec.make_input().view(np.int32)
    out = oracle.forward(spec, w, ids.view(np.uint8))
    cfg = BertConfig(vocab_size=1000, hidden_size=128, num_hidden_layers=2, num_attention_heads=2,
                     intermediate_size=256, max_position_embeddings=64, hidden_act="gelu",
                     layer_norm_eps=float(np.float32(1e-12)), hidden_dropout_prob=0.0,
                     attention_probs_dropout_prob=0.0, attn_implementation="eager")
    hf = BertForQuestionAnswering(cfg).double().eval()
    T = lambda n: torch.tensor(_t(w, spec, n))
    sd = {"bert.embeddings.word_embeddings.weight": T("embeddings.word"),
          "bert.embeddings.position_embeddings.weight": T("embeddings.position"),
          "bert.embeddings.token_type_embeddings.weight": T("embeddings.token_type"),
          "bert.embeddings.LayerNorm.weight": T("embeddings.ln.gamma"),
          "bert.embeddings.LayerNorm.bias": T("embeddings.ln.beta"),
          "qa_outputs.weight": T("qa.weight"), "qa_outputs.bias": T("qa.bias")}
    H = 128
    for i in range(2):
        p, q = f"bert.encoder.layer.{i}.", f"layer{i}."
        Wq, bq = T(q + "qkv.weight"), T(q + "qkv.bias")
        for j, nm in enumerate(["query", "key", "value"]):
            sd[p + f"attention.self.{nm}.weight"] = Wq[j * H:(j + 1) * H]
            sd[p + f"attention.self.{nm}.bias"] = bq[j * H:(j + 1) * H]
        sd[p + "attention.output.dense.weight"] = T(q + "attn_out.weight")
        sd[p + "attention.output.dense.bias"] = T(q + "attn_out.bias")
        sd[p + "attention.output.LayerNorm.weight"] = T(q + "ln1.gamma")
        sd[p + "attention.output.LayerNorm.bias"] = T(q + "ln1.beta")
        sd[p + "intermediate.dense.weight"] = T(q + "ffn1.weight")
        sd[p + "intermediate.dense.bias"] = T(q + "ffn1.bias")
        sd[p + "output.dense.weight"] = T(q + "ffn2.weight")
        sd[p + "output.dense.bias"] = T(q + "ffn2.bias")
        sd[p + "output.LayerNorm.weight"] = T(q + "ln2.gamma")
        sd[p + "output.LayerNorm.bias"] = T(q + "ln2.beta")
    missing, unexpected = hf.load_state_dict(sd, strict=False)
    assert not unexpected and all("position_ids" in k or "token_type_ids" in k for k in missing), missing
    with torch.no_grad():
        r = hf(input_ids=torch.tensor(ids[None].astype(np.int64)), token_type_ids=torch.zeros(1, 64, dtype=torch.long))
    logits = torch.stack([r.start_logits[0], r.end_logits[0]], dim=-1).numpy()
    np.testing.assert_allclose(out[spec.output_slot], logits, rtol=1e-10, atol=1e-11)
    # pooler: tanh(W_p x_0 + b_p) vs an independent float64 evaluation
    xs = out[[s.name for s in spec.slots].index("x")]
    pooled = np.tanh(T("pooler.weight").numpy() @ xs[0] + T("pooler.bias").numpy())
    np.testing.assert_allclose(out[[s.name for s in spec.slots].index("pooled")][0], pooled, rtol=1e-12)


def test_gpt2_tiny_vs_hf_transformers_float64():
    from transformers import GPT2Config, GPT2LMHeadModel
    spec = synth.build_model("gpt2-tiny")
    w = spec.build_weights()
    ids = spec.make_input().view(np.int32)
    y = oracle.output(spec, w, ids.view(np.uint8))
    cfg = GPT2Config(vocab_size=1000, n_positions=64, n_embd=128, n_layer=2, n_head=2,
                     activation_function="gelu_new", layer_norm_epsilon=float(np.float32(1e-5)),
                     resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0, attn_implementation="eager")
    hf = GPT2LMHeadModel(cfg).double().eval()
    T = lambda n: torch.tensor(_t(w, spec, n))
    sd = {"transformer.wte.weight": T("wte"), "transformer.wpe.weight": T("wpe"),
          "transformer.ln_f.weight": T("ln_f.gamma"), "transformer.ln_f.bias": T("ln_f.beta"),
          "lm_head.weight": T("wte")}
    for i in range(2):
        p, q = f"transformer.h.{i}.", f"h{i}."
        sd[p + "ln_1.weight"], sd[p + "ln_1.bias"] = T(q + "ln_1.gamma"), T(q + "ln_1.beta")
        sd[p + "ln_2.weight"], sd[p + "ln_2.bias"] = T(q + "ln_2.gamma"), T(q + "ln_2.beta")
        for nm in ["attn.c_attn", "attn.c_proj", "mlp.c_fc", "mlp.c_proj"]:
            sd[p + nm + ".weight"] = T(q + nm + ".weight").T.contiguous()   # HF Conv1D is [in, out]
            sd[p + nm + ".bias"] = T(q + nm + ".bias")
    hf.load_state_dict(sd, strict=False)
    with torch.no_grad():
        r = hf(input_ids=torch.tensor(ids[None].astype(np.int64)))
    np.testing.assert_allclose(y[0], r.logits[0, -1].numpy(), rtol=1e-10, atol=1e-11)


def test_resnet_tiny_vs_torch_functional_float64():
    spec = synth.build_model("resnet-tiny")
    w = spec.build_weights()
    img = spec.make_input()
    y = oracle.output(spec, w, img)
    vals = {spec.input_slot: torch.tensor(bf16_bits_to_f64(img.view(np.uint16)).reshape(spec.slots[0].shape))}
    for l in spec.layers:
        x = vals[l.in0]
        if l.op == Op.CONV2D:
            W = torch.tensor(_t(w, spec, spec.tensors[l.refs[0]].name)).permute(0, 3, 1, 2)
            b = torch.tensor(_t(w, spec, spec.tensors[l.refs[1]].name))
            o = F.conv2d(x.permute(2, 0, 1)[None], W, b, stride=l.attr[1], padding=l.attr[2])[0].permute(1, 2, 0)
            if l.in1 >= 0:
                o = o + vals[l.in1]
            if l.attr[0] == Act.RELU:
                o = torch.relu(o)
        elif l.op == Op.MAXPOOL:
            o = F.max_pool2d(x.permute(2, 0, 1)[None], l.attr[0], l.attr[1], l.attr[2])[0].permute(1, 2, 0)
        elif l.op == Op.AVGPOOL:
            o = x.mean(dim=(0, 1))[None]
        elif l.op == Op.LINEAR:
            o = F.linear(x, torch.tensor(_t(w, spec, spec.tensors[l.refs[0]].name)),
                         torch.tensor(_t(w, spec, spec.tensors[l.refs[1]].name)))
        vals[l.out] = o
    np.testing.assert_allclose(y, vals[spec.output_slot].numpy(), rtol=1e-11, atol=1e-11)


# ---------------------------------------------------------------------------------------------
# ResNet-50 v1.5 against torchvision (SURVEY §8(c) reading #5: BN folded, stride on the 3x3)
# ---------------------------------------------------------------------------------------------
def _tv_resnet50_folded(spec, seed=0):
    """torchvision's resnet50 (float64, eval) with random BatchNorm statistics; every conv+BN pair folded
    into (W', b') in float64, written into the synth table's tensors (bf16), and the rounded values
    loaded back into the torchvision model with each BN reduced to `+ b'` (var 1, mean 0,
    gamma 1; eps 1e-300 leaves sqrt(var + eps) == 1), so both sides compute with the same weights."""
    import torchvision
    torch.manual_seed(seed)
    tv = torchvision.models.resnet50(weights=None).double().eval()
    for m in tv.modules():
        if isinstance(m, torch.nn.BatchNorm2d):
            m.running_mean.uniform_(-0.1, 0.1)
            m.running_var.uniform_(0.5, 1.5)
            m.weight.data.uniform_(0.3, 0.6)
            m.bias.data.uniform_(-0.1, 0.1)
    pairs = [("conv1", tv.conv1, tv.bn1)]
    for si in range(4):
        for bi, blk in enumerate(getattr(tv, f"layer{si + 1}")):
            p = f"layer{si + 1}.{bi}"
            pairs += [(p + ".conv1", blk.conv1, blk.bn1), (p + ".conv2", blk.conv2, blk.bn2),
                      (p + ".conv3", blk.conv3, blk.bn3)]
            if blk.downsample is not None:
                pairs.append((p + ".downsample", blk.downsample[0], blk.downsample[1]))
    ov = {}
    with torch.no_grad():
        for name, conv, bn in pairs:
            s = bn.weight / torch.sqrt(bn.running_var + bn.eps)
            ov[name + ".weight"] = (conv.weight * s[:, None, None, None]).permute(0, 2, 3, 1).numpy()
            ov[name + ".bias"] = (bn.bias - bn.running_mean * s).numpy()
        ov["fc.weight"], ov["fc.bias"] = tv.fc.weight.numpy(), tv.fc.bias.numpy()
    w = spec.build_weights(ov)
    with torch.no_grad():
        for name, conv, bn in pairs:
            conv.weight.copy_(torch.tensor(_t(w, spec, name + ".weight")).permute(0, 3, 1, 2))
            bn.running_mean.zero_()
            bn.running_var.fill_(1.0)
            bn.eps = 1e-300  # sqrt(1 + eps) == 1 in float64
            bn.weight.fill_(1.0)
            bn.bias.copy_(torch.tensor(_t(w, spec, name + ".bias")))
        tv.fc.weight.copy_(torch.tensor(_t(w, spec, "fc.weight")))
        tv.fc.bias.copy_(torch.tensor(_t(w, spec, "fc.bias")))
    return tv, w


def _tv_input(spec, img):
    return torch.tensor(bf16_bits_to_f64(img.view(np.uint16)).reshape(spec.slots[spec.input_slot].shape)).permute(2, 0, 1)[None]


def test_resnet50_v15_table_vs_torchvision_float64():
    """The synth ResNet-50 table (reduced to a 64x64 image, full widths and depths) run by the oracle equals
    torchvision.models.resnet50 (v1.5) in float64 with the same folded weights.  Negative controls: the v1
    block (stride on the first 1x1) and ReLU before the residual add must NOT match."""
    spec = synth.models._resnet([3, 4, 6, 3], [64, 128, 256, 512], 64, name="resnet50-64px")
    tv, w = _tv_resnet50_folded(spec)
    img = spec.make_input()
    y = oracle.output(spec, w, img).reshape(-1)
    with torch.no_grad():
        ref = tv(_tv_input(spec, img))[0].numpy()
    assert np.max(np.abs(y - ref)) <= 1e-9 * np.max(np.abs(ref)), np.max(np.abs(y - ref))
    # v1: stride moved to the first 1x1 of each stage's first block
    with torch.no_grad():
        for si in (2, 3, 4):
            blk = getattr(tv, f"layer{si}")[0]
            blk.conv1.stride, blk.conv2.stride = (2, 2), (1, 1)
        v1 = tv(_tv_input(spec, img))[0].numpy()
        for si in (2, 3, 4):
            blk = getattr(tv, f"layer{si}")[0]
            blk.conv1.stride, blk.conv2.stride = (1, 1), (2, 2)
    assert np.max(np.abs(y - v1)) > 1e-3 * np.max(np.abs(ref))
    # ReLU applied to the conv3 branch before the residual add (instead of after the add)
    from torchvision.models.resnet import Bottleneck

    def relu_before_add(self, x):
        idt = x if self.downsample is None else self.downsample(x)
        o = self.relu(self.bn1(self.conv1(x)))
        o = self.relu(self.bn2(self.conv2(o)))
        return self.relu(self.bn3(self.conv3(o))) + idt
    orig = Bottleneck.forward
    Bottleneck.forward = relu_before_add
    try:
        with torch.no_grad():
            rb = tv(_tv_input(spec, img))[0].numpy()
    finally:
        Bottleneck.forward = orig
    assert np.max(np.abs(y - rb)) > 1e-3 * np.max(np.abs(ref))
