"""Per-op first-light parity on the GPU (debug aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
from synth.models import ModelSpec, Op, Act, DT_BF16, DT_F32, DT_I32, f32_bits, to_bf16_bits, bf16_bits_to_f64
from paper_2306_03622_b200 import Runtime

rt = Runtime(pool_bytes=2 << 30)

def run(spec, w, x, tag):
    mid = rt.register_spec(spec, w)
    outs = []
    for i in range(2):
        r = rt.invoke(mid, x)
        outs.append(r.output.copy())
    ref = oracle.output(spec, w, x).reshape(-1)
    got = outs[0].astype(np.float64).reshape(-1) if outs[0].dtype != np.uint16 else bf16_bits_to_f64(outs[0]).reshape(-1)
    got2 = outs[1].astype(np.float64).reshape(-1) if outs[1].dtype != np.uint16 else bf16_bits_to_f64(outs[1]).reshape(-1)
    err = np.abs(got - ref)
    rel = err.max() / max(1e-30, np.abs(ref).max())
    shape = spec.slots[spec.output_slot].shape
    bad = np.argwhere(err.reshape(shape) > 1e-2 * max(1e-30, np.abs(ref).max()))
    print(f"{tag}: rel={rel:.3e} det={np.array_equal(got, got2)} nbad={len(bad)} first_bad={bad[:6].tolist()}", flush=True)
    if len(bad):
        b = tuple(bad[0])
        print("   got", got.reshape(shape)[b], "ref", ref.reshape(shape)[b])
    return got.reshape(shape), ref.reshape(shape)

def linear(M, K, N, integer=True, out_dt=DT_F32, in_dt=DT_BF16, seed=0):
    m = ModelSpec(f"lin{M}x{K}x{N}", 5)
    xs = m.slot("x", (M, K), in_dt)
    ys = m.slot("y", (M, N), out_dt)
    w_ = m.tensor("w", (N, K)); b_ = m.tensor("b", (N,))
    m.layer(Op.LINEAR, [w_, b_], xs, -1, ys, [Act.NONE])
    m.input_slot, m.output_slot = xs, ys
    rng = np.random.default_rng(seed)
    if integer:
        W = rng.integers(-2, 3, (N, K)).astype(np.float64); B = rng.integers(-2, 3, N).astype(np.float64)
        X = rng.integers(-2, 3, (M, K)).astype(np.float64)
    else:
        W = rng.uniform(-0.05, 0.05, (N, K)); B = rng.uniform(-0.05, 0.05, N); X = rng.uniform(-1, 1, (M, K))
    w = m.build_weights({"w": W, "b": B})
    x = to_bf16_bits(X).view(np.uint8) if in_dt == DT_BF16 else X.astype(np.float32).view(np.uint8)
    return m, w, x

for (M, K, N) in [(128, 64, 16), (128, 64, 64), (128, 256, 64), (128, 768, 2304), (64, 128, 128), (300, 192, 96)]:
    m, w, x = linear(M, K, N)
    g, r = run(m, w, x, f"linear M{M} K{K} N{N} int")
    if M == 128 and K == 64 and N == 16:
        print("   row0 got", g[0, :8], "ref", r[0, :8])
        print("   row1 got", g[1, :8], "ref", r[1, :8])
        print("   row8 got", g[8, :8], "ref", r[8, :8])

# layernorm
m = ModelSpec("ln", 6); xs = m.slot("x", (128, 768), DT_F32); ys = m.slot("y", (128, 768), DT_F32)
g_ = m.tensor("g", (768,), init=("range", 0.9, 1.1)); b_ = m.tensor("b", (768,), init=("uniform", 0.05))
m.layer(Op.LAYERNORM, [g_, b_], xs, -1, ys, [f32_bits(1e-12)]); m.input_slot, m.output_slot = xs, ys
x = np.random.default_rng(1).standard_normal((128, 768)).astype(np.float32).view(np.uint8)
run(m, m.build_weights(), x, "layernorm")

# attention
for causal in (0, 1):
    m = ModelSpec("attn", 7); xs = m.slot("qkv", (128, 3 * 128), DT_BF16); ys = m.slot("ctx", (128, 128), DT_BF16)
    q2 = m.slot("qkv2", (128, 384), DT_BF16)
    w_ = m.tensor("w", (384, 384))
    m.layer(Op.LINEAR, [w_], xs, -1, q2, [Act.NONE])
    m.layer(Op.ATTENTION, [], q2, -1, ys, [2, 64, causal]); m.input_slot, m.output_slot = xs, ys
    x = to_bf16_bits(np.random.default_rng(2).standard_normal((128, 384))).view(np.uint8)
    try:
        run(m, m.build_weights({"w": np.eye(384)}), x, f"attention causal={causal}")
    except Exception as e:
        print("attention", e)
rt.close()
