"""GPU parity: libfsw's cold swap-in-and-execute vs the CPU oracle (float64) on the same seeded
weights and inputs.  Bar: max|gpu − ref| ≤ 1e-2·max|ref| over every output element (BASELINE.json
north_star); bit-exact where the arithmetic is exact (integer MLPs, closed forms)."""
import numpy as np
import pytest

import oracle
import synth
from synth.models import Act, bf16_bits_to_f64

pytestmark = pytest.mark.gpu

TOL = 1e-2


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    return float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))


@pytest.mark.parametrize("name", ["mlp-small", "mlp", "bert-tiny", "gpt2-tiny", "resnet-tiny",
                                  "bert-base", "resnet50", "gpt2-2L",
                                  "resnet101", "resnet152", "bert-large"])  # + the paper's other models
def test_cold_invoke_matches_oracle(rt, registered, name):
    spec, w, x, mid = registered(name)
    rt.evict(mid)
    r = rt.invoke(mid, x, gpu=0)
    ref = oracle.output(spec, w, x)
    assert np.all(np.isfinite(r.output))
    assert rel_err(r.output, ref) <= TOL


def test_gpt2_xl_full_matches_oracle(rt):
    spec = synth.build_model("gpt2-xl")
    w = spec.build_weights()
    x = spec.make_input()
    mid = rt.register_spec(spec, w)
    try:
        r = rt.invoke(mid, x, gpu=0)
        # the whole 3.1 GB extent, every byte (the extent was poisoned before the swap)
        assert np.array_equal(rt.read_resident(mid, 0), rt.read_store(mid))
        assert rel_err(r.output, oracle.output(spec, w, x)) <= TOL
    finally:
        rt.unregister(mid)


def _integer_mlp(width, seed):
    spec = synth.mlp(width=width, n_layers=4, act=Act.RELU, seed=seed)
    rng = np.random.default_rng(seed)
    ov = {}
    for l in spec.layers:
        wt, bt = spec.tensors[l.refs[0]], spec.tensors[l.refs[1]]
        W = np.zeros(wt.shape)
        for o in range(wt.shape[0]):
            cols = rng.choice(wt.shape[1], size=4, replace=False)
            W[o, cols] = rng.choice([-1.0, 1.0], size=4)
        ov[wt.name], ov[bt.name] = W, rng.integers(-1, 2, wt.shape[0]).astype(np.float64)
    x = rng.integers(-1, 2, (1, width)).astype(np.float32)
    return spec, ov, x


@pytest.mark.parametrize("width,seed", [(1024, 21), (1024, 22), (256, 23)])
def test_integer_mlp_bit_exact(rt, width, seed):
    """sparse ±1 weights, {−1,0,1} inputs/biases keep every intermediate an exact
    integer ≤ 256 in bf16, so GPU == oracle == int64 brute force bit-exactly."""
    spec, ov, x = _integer_mlp(width, seed)
    w = spec.build_weights(ov)
    mid = rt.register_spec(spec, w)
    try:
        r = rt.invoke(mid, x.view(np.uint8), gpu=0)
        h = x.astype(np.int64)
        for i, l in enumerate(spec.layers):
            h = h @ ov[spec.tensors[l.refs[0]].name].astype(np.int64).T + ov[spec.tensors[l.refs[1]].name].astype(np.int64)
            if i < 3:
                h = np.maximum(h, 0)
        np.testing.assert_array_equal(r.output.reshape(1, -1), h.astype(np.float32))
        np.testing.assert_array_equal(r.output.reshape(1, -1), oracle.output(spec, w, x.view(np.uint8)))
    finally:
        rt.unregister(mid)


def test_integer_gemm_path_bit_exact(rt):
    """The tcgen05 GEMM path (M = 128 rows) on exact small-integer data: bit-exact vs int64."""
    from synth.models import DT_BF16, DT_F32, ModelSpec, Op, to_bf16_bits
    rng = np.random.default_rng(5)
    for (M, K, N) in [(128, 768, 2304), (300, 192, 96), (49, 4608, 512), (128, 1600, 4800)]:
        m = ModelSpec("intgemm", 5)
        xs = m.slot("x", (M, K), DT_BF16)
        ys = m.slot("y", (M, N), DT_F32)
        w_, b_ = m.tensor("w", (N, K)), m.tensor("b", (N,))
        m.layer(Op.LINEAR, [w_, b_], xs, -1, ys, [Act.NONE])
        m.input_slot, m.output_slot = xs, ys
        W = rng.integers(-2, 3, (N, K)); B = rng.integers(-2, 3, N); X = rng.integers(-2, 3, (M, K))
        w = m.build_weights({"w": W.astype(np.float64), "b": B.astype(np.float64)})
        mid = rt.register_spec(m, w)
        try:
            r = rt.invoke(mid, to_bf16_bits(X.astype(np.float64)).view(np.uint8), gpu=0)
            np.testing.assert_array_equal(r.output.reshape(M, N), (X @ W.T + B).astype(np.float32))
        finally:
            rt.unregister(mid)


def test_mlp_closed_forms(rt):
    n = 1024
    spec = synth.mlp(width=n, n_layers=4, act=Act.RELU, seed=3)
    x = np.linspace(-1, 1, n, dtype=np.float32).reshape(1, n)
    ov = {}
    for l in spec.layers:
        ov[spec.tensors[l.refs[0]].name] = np.eye(n)
        ov[spec.tensors[l.refs[1]].name] = np.zeros(n)
    mid = rt.register_spec(spec, spec.build_weights(ov))
    try:
        y = rt.invoke(mid, x.view(np.uint8), gpu=0).output.reshape(1, n)
        # W = I, b = 0: y = relu(relu(relu(x))) stored through bf16 hidden slots
        np.testing.assert_array_equal(y, bf16_bits_to_f64(synth.models.to_bf16_bits(np.maximum(x, 0))).reshape(1, n))
    finally:
        rt.unregister(mid)
    bias = np.arange(n) * 0.25 - 3
    for l in spec.layers:
        ov[spec.tensors[l.refs[0]].name] = np.zeros((n, n))
    ov[spec.tensors[spec.layers[-1].refs[1]].name] = bias
    mid = rt.register_spec(spec, spec.build_weights(ov))
    try:
        y = rt.invoke(mid, x.view(np.uint8), gpu=0).output
        # all W = 0 ⇒ y = b4 exactly, b4 as stored: bf16 (DESIGN.md §3 reading 1); 252.25 etc.
        # are not bf16 values, so the closed form is the RNE-rounded bias
        b4 = bf16_bits_to_f64(synth.models.to_bf16_bits(bias)).astype(np.float32)
        np.testing.assert_array_equal(y.reshape(-1), b4)
    finally:
        rt.unregister(mid)


def _zero_linears(spec):
    ov = {}
    for l in spec.layers:
        if l.op in (3, 5):
            for r in l.refs:
                t = spec.tensors[r]
                if t.name not in ("wte", "qa.bias", "fc.bias"):
                    ov[t.name] = np.zeros(t.shape)
    return ov


@pytest.mark.parametrize("name", ["bert-base", "resnet50"])
def test_zero_linear_networks_closed_form(rt, name):
    """All Linear/conv W,b = 0 ⇒ BERT QA logits = b_qa, ResNet logits = fc bias, exactly."""
    spec = synth.build_model(name)
    w = spec.build_weights(_zero_linears(spec))
    mid = rt.register_spec(spec, w)
    try:
        y = rt.invoke(mid, spec.make_input(), gpu=0).output
        bname = "qa.bias" if name == "bert-base" else "fc.bias"
        t = spec.tensors[spec.tensor_index(bname)]
        b = bf16_bits_to_f64(w[t.offset:t.offset + t.nbytes].view(np.uint16))
        n_rows = y.size // b.size
        np.testing.assert_array_equal(y.reshape(n_rows, -1), np.broadcast_to(b, (n_rows, b.size)).astype(np.float32))
    finally:
        rt.unregister(mid)


def test_bert_pooler_and_hidden_slots(rt, registered):
    spec, w, x, mid = registered("bert-base")
    rt.evict(mid)
    rt.invoke(mid, x, gpu=0)
    ref = oracle.forward(spec, w, x)
    names = [s.name for s in spec.slots]
    for nm in ("pooled", "x"):
        sid = names.index(nm)
        got = rt.read_slot(mid, sid, spec.slots[sid].nbytes).view(np.float32)
        assert rel_err(got, ref[sid]) <= TOL, nm


def test_gpt_causal_mask_prefix_mean(rt):
    """W_q = W_k = 0 in every layer's c_attn ⇒ uniform causal softmax ⇒ ctx row t = prefix mean of v.
    Checked on the layer-0 attention output slot against the float64 prefix mean of the GPU's own qkv."""
    spec = synth.build_model("gpt2-tiny")
    H = 128
    ov = {}
    w0 = spec.build_weights()
    for l in spec.layers:
        if l.name.endswith("c_attn"):
            t = spec.tensors[l.refs[0]]
            W = bf16_bits_to_f64(w0[t.offset:t.offset + t.nbytes].view(np.uint16)).reshape(t.shape).copy()
            W[:2 * H] = 0
            ov[t.name] = W
            bt = spec.tensors[l.refs[1]]
            Bv = bf16_bits_to_f64(w0[bt.offset:bt.offset + bt.nbytes].view(np.uint16)).copy()
            Bv[:2 * H] = 0
            ov[bt.name] = Bv
    w = spec.build_weights(ov)
    mid = rt.register_spec(spec, w)
    try:
        rt.invoke(mid, spec.make_input(), gpu=0)
        names = [s.name for s in spec.slots]
        qkv = bf16_bits_to_f64(rt.read_slot(mid, names.index("qkv"), 64 * 3 * H * 2).view(np.uint16)).reshape(64, 3 * H)
        ctx = bf16_bits_to_f64(rt.read_slot(mid, names.index("ctx"), 64 * H * 2).view(np.uint16)).reshape(64, H)
        v = qkv[:, 2 * H:]
        ref = np.cumsum(v, axis=0) / np.arange(1, 65)[:, None]
        np.testing.assert_allclose(ctx, ref, rtol=1e-2, atol=1e-2 * np.abs(ref).max())
    finally:
        rt.unregister(mid)
