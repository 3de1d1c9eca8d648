"""Per-GEMM time inside a dependent chain, libfsw vs cuBLAS, at BERT-base's batch-1 linear shapes (VERDICT r1 #3:
"in-graph BERT QKV / FFN1 / FFN2 each <= 1.2x cuBLAS").

libfsw: a synthetic model of 12 linears of one shape (x -> y_1, y_1 -> y_2 when the shape chains, else all from
x), resident, one invoke = one CUDA graph of 12 dependent GEMM launches (PDL chain); per-GEMM = invoke time / 12
(includes the model's embed-free graph overhead: measured separately with a 1-linear model and subtracted).
cuBLAS: the same 12 F.linear calls (distinct bf16 weights, bias, GELU where the BERT layer has it) in a torch
CUDA graph, two weight copies replayed alternately (weights from HBM as in libfsw).

    python tools/gemm_chain_vs_cublas.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2306_03622_b200 import Runtime  # noqa: E402
from synth.models import DT_BF16, Act, ModelSpec, Op  # noqa: E402

T = 128
SHAPES = {"qkv": (768, 2304, Act.NONE), "o-proj": (768, 768, Act.NONE), "ffn1": (768, 3072, Act.GELU_ERF),
          "ffn2": (3072, 768, Act.NONE),
          # GPT-2-XL's (run only when named on the command line)
          "gpt-qkv": (1600, 4800, Act.NONE), "gpt-proj": (1600, 1600, Act.NONE), "gpt-fc": (1600, 6400, Act.GELU_TANH),
          "gpt-proj2": (6400, 1600, Act.NONE)}
DEFAULT = ["qkv", "o-proj", "ffn1", "ffn2"]
N_CHAIN = 12


def chain_model(K, N, act, n):
    m = ModelSpec(f"chain{K}x{N}x{n}", 7, input_kind=("uniform_bf16", 1.0))
    x = m.slot("x", (T, K), DT_BF16)
    prev = x
    for i in range(n):
        w = m.tensor(f"w{i}", (N, K), init=("uniform", (3.0 / K) ** 0.5))
        b = m.tensor(f"b{i}", (N,), init=("uniform", 0.1))
        out = m.slot(f"y{i}", (T, N), DT_BF16)
        m.layer(Op.LINEAR, [w, b], in0=prev if K == N else x, out=out, attr=[int(act), 0, 0], name=f"l{i}")
        prev = out
    m.input_slot, m.output_slot = x, prev
    return m


def fsw_resident_ms(rt, spec, reps=200):
    w, x = spec.build_weights(), spec.make_input()
    mid = rt.register_spec(spec, w)
    for _ in range(20):
        rt.invoke(mid, x, gpu=0)
    t = sorted(rt.invoke(mid, x, gpu=0).stats["device_ms"] for _ in range(reps))
    rt.unregister(mid)
    return t[len(t) // 2]


def cublas_chain_ms(K, N, act, n, reps=200):
    dev = "cuda"
    mk = lambda: [((torch.randn(N, K, device=dev) * (3.0 / K) ** 0.5).to(torch.bfloat16),
                   (torch.randn(N, device=dev) * 0.1).to(torch.bfloat16)) for _ in range(n)]
    wa, wb = mk(), mk()
    x = torch.randn(T, K, device=dev).to(torch.bfloat16)

    def run(ws):
        h = x
        for w, b in ws:
            y = F.linear(h if K == N else x, w, b)
            h = F.gelu(y) if act == Act.GELU_ERF else F.gelu(y, approximate="tanh") if act == Act.GELU_TANH else y
        return h

    ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run(wa), run(wb)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(ga):
        run(wa)
    with torch.cuda.graph(gb):
        run(wb)
    for _ in range(20):
        ga.replay(), gb.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2 * reps)]
    for i in range(reps):
        for k, g in enumerate((ga, gb)):
            e0, e1 = ev[2 * i + k]
            e0.record()
            g.replay()
            e1.record()
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    return t[len(t) // 2]


def main():
    only = [a for a in sys.argv[1:] if a in SHAPES] or DEFAULT
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FSW_"))
    with torch.inference_mode(), Runtime(gpu_ids=[0], pool_bytes=4 << 30) as rt:
        for name, (K, N, act) in SHAPES.items():
            if only and name not in only:
                continue
            f12 = fsw_resident_ms(rt, chain_model(K, N, act, N_CHAIN))
            f1 = fsw_resident_ms(rt, chain_model(K, N, act, 1))
            c12 = cublas_chain_ms(K, N, act, N_CHAIN)
            c1 = cublas_chain_ms(K, N, act, 1)
            fg, cg = (f12 - f1) / (N_CHAIN - 1) * 1e3, (c12 - c1) / (N_CHAIN - 1) * 1e3
            print(f"[{tag}] {name:7s} M={T} K={K} N={N}: libfsw {fg:6.2f} us per GEMM in the chain, cuBLAS {cg:6.2f} us "
                  f"-> ratio {fg / cg:.2f} (chains of 12: {f12 * 1e3:.1f} / {c12 * 1e3:.1f} us)", flush=True)


if __name__ == "__main__":
    main()
