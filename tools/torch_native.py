"""Context row of SURVEY §8(d) protocol step 2: the same model shapes run as a plain PyTorch bf16 forward (cuBLAS
GEMMs, SDPA attention, native LayerNorm / GELU) captured in a CUDA graph, resident in HBM — the analogue of the
paper's "Native" column.  Bench-only, never a product path: it shares nothing with libfsw.

Each replay runs with the weights of one of two model copies (together larger than the 126-MB L2), alternating,
so weights come from HBM as in a resident libfsw invoke after other traffic.

    python tools/torch_native.py [bert-base resnet50 gpt2-xl]
"""
import sys

import torch
import torch.nn.functional as F


def bert_base(dev):
    H, FF, L, V = 768, 3072, 12, 30522
    r = lambda *s: (torch.randn(*s, device=dev) * 0.02).to(torch.bfloat16)
    p = {"word": r(V, H), "pos": r(512, H), "type": r(2, H), "ln_g": torch.ones(H, device=dev), "ln_b": torch.zeros(H, device=dev),
         "layers": [], "pool_w": r(H, H), "pool_b": r(H), "qa_w": r(2, H), "qa_b": r(2)}
    for _ in range(L):
        p["layers"].append({"qkv_w": r(3 * H, H), "qkv_b": r(3 * H), "o_w": r(H, H), "o_b": r(H),
                            "ln1_g": torch.ones(H, device=dev), "ln1_b": torch.zeros(H, device=dev),
                            "f1_w": r(FF, H), "f1_b": r(FF), "f2_w": r(H, FF), "f2_b": r(H),
                            "ln2_g": torch.ones(H, device=dev), "ln2_b": torch.zeros(H, device=dev)})
    return p


def bert_forward(p, ids):
    T, H = ids.shape[0], 768
    x = (p["word"][ids].float() + p["pos"][:T].float() + p["type"][0].float())
    x = F.layer_norm(x, (H,), p["ln_g"], p["ln_b"], 1e-12)
    for lp in p["layers"]:
        xb = x.to(torch.bfloat16)
        qkv = F.linear(xb, lp["qkv_w"], lp["qkv_b"]).view(T, 3, 12, 64).permute(1, 2, 0, 3)
        a = F.scaled_dot_product_attention(qkv[0][None], qkv[1][None], qkv[2][None])[0].permute(1, 0, 2).reshape(T, H)
        x = F.layer_norm(x + F.linear(a, lp["o_w"], lp["o_b"]).float(), (H,), lp["ln1_g"], lp["ln1_b"], 1e-12)
        h = F.gelu(F.linear(x.to(torch.bfloat16), lp["f1_w"], lp["f1_b"]))
        x = F.layer_norm(x + F.linear(h, lp["f2_w"], lp["f2_b"]).float(), (H,), lp["ln2_g"], lp["ln2_b"], 1e-12)
    xb = x.to(torch.bfloat16)
    pooled = torch.tanh(F.linear(xb[:1], p["pool_w"], p["pool_b"]))
    return F.linear(xb, p["qa_w"], p["qa_b"]).float(), pooled


def gpt2_xl(dev):
    H, L, V = 1600, 48, 50257
    r = lambda *s: (torch.randn(*s, device=dev) * 0.02).to(torch.bfloat16)
    p = {"wte": r(V, H), "wpe": r(1024, H), "lnf_g": torch.ones(H, device=dev), "lnf_b": torch.zeros(H, device=dev), "layers": []}
    for _ in range(L):
        p["layers"].append({"ln1_g": torch.ones(H, device=dev), "ln1_b": torch.zeros(H, device=dev),
                            "qkv_w": r(3 * H, H), "qkv_b": r(3 * H), "o_w": r(H, H), "o_b": r(H),
                            "ln2_g": torch.ones(H, device=dev), "ln2_b": torch.zeros(H, device=dev),
                            "fc_w": r(4 * H, H), "fc_b": r(4 * H), "p2_w": r(H, 4 * H), "p2_b": r(H)})
    return p


def gpt2_forward(p, ids):
    T, H = ids.shape[0], 1600
    x = p["wte"][ids].float() + p["wpe"][:T].float()
    for lp in p["layers"]:
        h = F.layer_norm(x, (H,), lp["ln1_g"], lp["ln1_b"], 1e-5).to(torch.bfloat16)
        qkv = F.linear(h, lp["qkv_w"], lp["qkv_b"]).view(T, 3, 25, 64).permute(1, 2, 0, 3)
        a = F.scaled_dot_product_attention(qkv[0][None], qkv[1][None], qkv[2][None], is_causal=True)[0].permute(1, 0, 2).reshape(T, H)
        x = x + F.linear(a, lp["o_w"], lp["o_b"]).float()
        h = F.layer_norm(x, (H,), lp["ln2_g"], lp["ln2_b"], 1e-5).to(torch.bfloat16)
        x = x + F.linear(F.gelu(F.linear(h, lp["fc_w"], lp["fc_b"]), approximate="tanh"), lp["p2_w"], lp["p2_b"]).float()
    h = F.layer_norm(x[-1:], (H,), p["lnf_g"], p["lnf_b"], 1e-5).to(torch.bfloat16)
    return F.linear(h, p["wte"]).float()


def resnet50(dev):
    import torchvision
    m = torchvision.models.resnet50().eval().to(dev).to(torch.bfloat16).to(memory_format=torch.channels_last)
    return m


def timed(fn_a, fn_b, reps):
    """Median replay time (ms) of two captured graphs (two weight copies) alternating."""
    ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn_a(), fn_b()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(ga):
        fn_a()
    with torch.cuda.graph(gb):
        fn_b()
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


def main(names=None, verbose=True):
    """{model: median replay ms}; prints a line per model when verbose (bench.py calls it quietly: its stdout is
    the one JSON line)."""
    dev = "cuda"
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = True
    names = names or sys.argv[1:] or ["bert-base", "resnet50", "gpt2-xl"]
    out = {}
    with torch.inference_mode():
        for name in names:
            if name == "bert-base":
                pa, pb = bert_base(dev), bert_base(dev)
                ids = torch.randint(0, 30522, (128,), device=dev)
                t = timed(lambda: bert_forward(pa, ids), lambda: bert_forward(pb, ids), 100)
            elif name == "gpt2-xl":
                pa, pb = gpt2_xl(dev), gpt2_xl(dev)
                ids = torch.randint(0, 50257, (128,), device=dev)
                t = timed(lambda: gpt2_forward(pa, ids), lambda: gpt2_forward(pb, ids), 20)
            else:
                ma, mb = resnet50(dev), resnet50(dev)
                x = torch.randn(1, 3, 224, 224, device=dev).to(torch.bfloat16).to(memory_format=torch.channels_last)
                t = timed(lambda: ma(x), lambda: mb(x), 100)
            out[name] = round(t, 4)
            if verbose:
                print(f"torch bf16 native (CUDA graph, weights from HBM) {name}: {t:.4f} ms", flush=True)
    return out


if __name__ == "__main__":
    main()
