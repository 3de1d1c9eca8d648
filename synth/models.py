"""Model descriptions (layer tables) and seeded weight/input generation.

A model is described the way the library's C-ABI receives it (include/fsw.h):
an ordered list of tensors (the caller's weight blob, row-major, execution
order), activation *slots* (named buffers), and layers in execution order.  The
paper records each function's parameter access pattern during its first run and
swaps in that order (§"Model Swapping"); the layer table here
is that access pattern written down explicitly, and execution order is swap
order ("executed layer by layer").

The four workload classes follow BASELINE.json ``configs`` and SURVEY §8(a):
tiny 4x1024 MLP, BERT-base (seq 128, QA head), ResNet-50 v1.5 (BN folded),
GPT-2-XL (seq 128, tied LM head on the last token).  Weights are random
(SURVEY §8c reading #14); the paper's trained weights are out of scope.

Nothing in this file computes a forward pass.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")


def build_lib(force: bool = False) -> str:
    src = os.path.join(_HERE, "csrc", "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
        u64, dbl, i32 = ctypes.c_uint64, ctypes.c_double, ctypes.c_int32
        vp = ctypes.c_void_p
        _lib.synth_uniform_bf16.argtypes = [vp, u64, u64, u64, dbl, dbl]
        _lib.synth_uniform_f32.argtypes = [vp, u64, u64, u64, dbl, dbl]
        _lib.synth_ids_i32.argtypes = [vp, u64, u64, u64, i32]
        _lib.synth_int_bf16.argtypes = [vp, u64, u64, u64, i32, i32]
        _lib.synth_normal_bf16.argtypes = [vp, u64, u64, u64, dbl]
        _lib.synth_laplace_bf16.argtypes = [vp, u64, u64, u64, dbl]
        for f in (_lib.synth_uniform_bf16, _lib.synth_uniform_f32, _lib.synth_ids_i32, _lib.synth_int_bf16,
                  _lib.synth_normal_bf16, _lib.synth_laplace_bf16):
            f.restype = None
    return _lib


# ----------------------------------------------------------------------------
# Table vocabulary (mirrors include/fsw.h)
# ----------------------------------------------------------------------------
class Op(IntEnum):
    EMBED = 1
    LAYERNORM = 2
    LINEAR = 3
    ATTENTION = 4
    CONV2D = 5
    MAXPOOL = 6
    AVGPOOL = 7


class Act(IntEnum):
    NONE = 0
    RELU = 1
    GELU_ERF = 2
    GELU_TANH = 3
    TANH = 4


class Rule(IntEnum):  # EMBED index rule per table
    IDS = 0        # row = input id of token t
    POSITION = 1   # row = t
    ZERO = 2       # row = 0 (BERT token type 0)


DT_BF16, DT_F32, DT_I32 = 0, 1, 2
DT_NAMES = {"bf16": DT_BF16, "f32": DT_F32, "i32": DT_I32}
DT_SIZE = {DT_BF16: 2, DT_F32: 4, DT_I32: 4}
ALIGN = 256  # tensor alignment in the caller's blob


def f32_bits(x: float) -> int:
    return int(np.array([x], dtype=np.float32).view(np.int32)[0])


@dataclass
class Tensor:
    name: str
    shape: tuple
    dtype: int = DT_BF16
    init: tuple = ("uniform", 0.0)  # ("uniform", bound) | ("range", lo, hi) | ("zeros",) | ("ones",)
    offset: int = 0

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape))

    @property
    def nbytes(self) -> int:
        return self.numel * DT_SIZE[self.dtype]


@dataclass
class Slot:
    name: str
    shape: tuple
    dtype: int = DT_BF16

    @property
    def nbytes(self) -> int:
        return int(np.prod(self.shape)) * DT_SIZE[self.dtype]


@dataclass
class Layer:
    op: int
    refs: List[int]
    in0: int = -1
    in1: int = -1
    out: int = -1
    attr: List[int] = field(default_factory=lambda: [0] * 8)
    name: str = ""


@dataclass
class ModelSpec:
    name: str
    seed: int
    tensors: List[Tensor] = field(default_factory=list)
    slots: List[Slot] = field(default_factory=list)
    layers: List[Layer] = field(default_factory=list)
    input_slot: int = 0
    output_slot: int = -1
    input_kind: tuple = ("uniform_f32", 1.0)
    # distribution of the ("uniform", a) bf16 tensors: "uniform" (U(±a), the default), or "gaussian" /
    # "laplace" with the same standard deviation a/√3 (bench: link coding on bell-shaped weights)
    dist: str = "uniform"

    # -- construction helpers ------------------------------------------------
    def tensor(self, name, shape, dtype=DT_BF16, init=("uniform", 0.02)) -> int:
        self.tensors.append(Tensor(name, tuple(shape), dtype, init))
        return len(self.tensors) - 1

    def slot(self, name, shape, dtype=DT_BF16) -> int:
        self.slots.append(Slot(name, tuple(shape), dtype))
        return len(self.slots) - 1

    def layer(self, op, refs, in0=-1, in1=-1, out=-1, attr=(), name="") -> int:
        a = list(attr) + [0] * (8 - len(attr))
        self.layers.append(Layer(int(op), list(refs), in0, in1, out, a, name))
        return len(self.layers) - 1

    # -- layout of the caller's blob ---------------------------------------------
    def assign_offsets(self) -> int:
        off = 0
        for t in self.tensors:
            t.offset = off
            off += (t.nbytes + ALIGN - 1) // ALIGN * ALIGN
        return off

    @property
    def weight_bytes(self) -> int:
        return self.assign_offsets()

    @property
    def param_count(self) -> int:
        return sum(t.numel for t in self.tensors)

    @property
    def algorithmic_bytes(self) -> int:
        return sum(t.nbytes for t in self.tensors)

    @property
    def input_bytes(self) -> int:
        return self.slots[self.input_slot].nbytes

    @property
    def output_bytes(self) -> int:
        return self.slots[self.output_slot].nbytes

    # -- generation --------------------------------------------------------------
    def build_weights(self, overrides: Optional[Dict[str, np.ndarray]] = None) -> np.ndarray:
        """Return the caller's weight blob (uint8), tensors row-major in execution order."""
        total = self.assign_offsets()
        blob = np.zeros(total, dtype=np.uint8)
        L = lib()
        for tid, t in enumerate(self.tensors):
            view = blob[t.offset:t.offset + t.nbytes]
            if overrides and t.name in overrides:
                arr = np.ascontiguousarray(overrides[t.name])
                if t.dtype == DT_BF16:
                    arr = to_bf16_bits(arr)
                elif t.dtype == DT_F32:
                    arr = arr.astype(np.float32)
                assert arr.size == t.numel, (t.name, arr.shape, t.shape)
                view[:] = arr.view(np.uint8).reshape(-1)
                continue
            kind = t.init[0]
            if kind in ("zeros",):
                continue
            if kind == "ones":
                lo = hi = 1.0
            elif kind == "uniform":
                lo, hi = -t.init[1], t.init[1]
            elif kind == "range":
                lo, hi = t.init[1], t.init[2]
            else:
                raise ValueError(kind)
            ptr = view.ctypes.data
            if t.dtype == DT_BF16 and kind == "uniform" and self.dist != "uniform":
                sigma = t.init[1] / math.sqrt(3.0)
                gen = {"gaussian": L.synth_normal_bf16, "laplace": L.synth_laplace_bf16}[self.dist]
                gen(ptr, t.numel, self.seed, tid + 1, sigma)
            elif t.dtype == DT_BF16:
                L.synth_uniform_bf16(ptr, t.numel, self.seed, tid + 1, lo, hi)
            elif t.dtype == DT_F32:
                L.synth_uniform_f32(ptr, t.numel, self.seed, tid + 1, lo, hi)
            else:
                raise ValueError("weights must be bf16 or f32")
        return blob

    def make_input(self, seed: Optional[int] = None) -> np.ndarray:
        """Return the request input bytes for the input slot (uint8 view)."""
        s = self.slots[self.input_slot]
        seed = self.seed * 1000 + 7 if seed is None else seed
        n = int(np.prod(s.shape))
        kind = self.input_kind
        if kind[0] == "ids":
            out = np.empty(n, dtype=np.int32)
            lib().synth_ids_i32(out.ctypes.data, n, seed, 0, kind[1])
        elif kind[0] == "uniform_f32":
            out = np.empty(n, dtype=np.float32)
            lib().synth_uniform_f32(out.ctypes.data, n, seed, 0, -kind[1], kind[1])
        elif kind[0] == "uniform_bf16":
            out = np.empty(n, dtype=np.uint16)
            lib().synth_uniform_bf16(out.ctypes.data, n, seed, 0, -kind[1], kind[1])
        else:
            raise ValueError(kind)
        assert out.nbytes == s.nbytes
        return out.view(np.uint8)

    def tensor_index(self, name: str) -> int:
        for i, t in enumerate(self.tensors):
            if t.name == name:
                return i
        raise KeyError(name)


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float array -> uint16 bf16 bit patterns, round-to-nearest-even."""
    f = np.ascontiguousarray(a, dtype=np.float32).reshape(-1)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return b.astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


# ----------------------------------------------------------------------------
# Workload classes
# ----------------------------------------------------------------------------
def mlp(width: int = 1024, n_layers: int = 4, act: int = Act.GELU_ERF, seed: int = 1,
        hidden_dtype: int = DT_BF16) -> ModelSpec:
    """BASELINE.json configs[0]: tiny MLP, batch 1.  h_i = act(W_i h_{i-1} + b_i); last layer linear."""
    m = ModelSpec(f"mlp{n_layers}x{width}", seed, input_kind=("uniform_f32", 1.0))
    x = m.slot("x", (1, width), DT_F32)
    prev = x
    he = math.sqrt(3.0) * math.sqrt(2.0 / width)
    for i in range(n_layers):
        w = m.tensor(f"fc{i}.weight", (width, width), init=("uniform", he))
        b = m.tensor(f"fc{i}.bias", (width,), init=("uniform", 0.05))
        last = i == n_layers - 1
        out = m.slot(f"h{i + 1}" if not last else "y", (1, width), DT_F32 if last else hidden_dtype)
        m.layer(Op.LINEAR, [w, b], in0=prev, out=out, attr=[Act.NONE if last else int(act), 0, 0], name=f"fc{i}")
        prev = out
    m.input_slot, m.output_slot = x, prev
    return m


def bert(n_layers=12, hidden=768, heads=12, inter=3072, vocab=30522, max_pos=512, seq=128,
         seed=2, name=None) -> ModelSpec:
    """BERT-base uncased encoder + pooler + QA head (SURVEY §8a a6, §8c oracle row 'BERT-base')."""
    m = ModelSpec(name or f"bert-L{n_layers}-H{hidden}", seed, input_kind=("ids", vocab))
    s = math.sqrt(3.0) * 0.02
    ids = m.slot("ids", (seq,), DT_I32)
    emb = m.slot("emb", (seq, hidden), DT_F32)
    x = m.slot("x", (seq, hidden), DT_F32)
    qkv = m.slot("qkv", (seq, 3 * hidden), DT_BF16)
    ctx = m.slot("ctx", (seq, hidden), DT_BF16)
    a = m.slot("attn_out", (seq, hidden), DT_F32)
    h = m.slot("h", (seq, hidden), DT_F32)
    f = m.slot("ffn", (seq, inter), DT_BF16)
    a2 = m.slot("ffn_out", (seq, hidden), DT_F32)
    pooled = m.slot("pooled", (1, hidden), DT_F32)
    logits = m.slot("qa_logits", (seq, 2), DT_F32)
    eps12 = f32_bits(1e-12)

    word = m.tensor("embeddings.word", (vocab, hidden), init=("uniform", s))
    pos = m.tensor("embeddings.position", (max_pos, hidden), init=("uniform", s))
    typ = m.tensor("embeddings.token_type", (2, hidden), init=("uniform", s))
    m.layer(Op.EMBED, [word, pos, typ], in0=ids, out=emb, attr=[3, Rule.IDS, Rule.POSITION, Rule.ZERO], name="embed")
    g = m.tensor("embeddings.ln.gamma", (hidden,), init=("range", 0.9, 1.1))
    bta = m.tensor("embeddings.ln.beta", (hidden,), init=("uniform", 0.05))
    m.layer(Op.LAYERNORM, [g, bta], in0=emb, out=x, attr=[eps12], name="embed_ln")
    dh = hidden // heads
    for i in range(n_layers):
        p = f"layer{i}."
        wq = m.tensor(p + "qkv.weight", (3 * hidden, hidden), init=("uniform", s))
        bq = m.tensor(p + "qkv.bias", (3 * hidden,), init=("uniform", s))
        m.layer(Op.LINEAR, [wq, bq], in0=x, out=qkv, attr=[Act.NONE], name=p + "qkv")
        m.layer(Op.ATTENTION, [], in0=qkv, out=ctx, attr=[heads, dh, 0], name=p + "attn")
        wo = m.tensor(p + "attn_out.weight", (hidden, hidden), init=("uniform", s))
        bo = m.tensor(p + "attn_out.bias", (hidden,), init=("uniform", s))
        m.layer(Op.LINEAR, [wo, bo], in0=ctx, in1=x, out=a, attr=[Act.NONE], name=p + "attn_out")
        g1 = m.tensor(p + "ln1.gamma", (hidden,), init=("range", 0.9, 1.1))
        b1 = m.tensor(p + "ln1.beta", (hidden,), init=("uniform", 0.05))
        m.layer(Op.LAYERNORM, [g1, b1], in0=a, out=h, attr=[eps12], name=p + "ln1")
        w1 = m.tensor(p + "ffn1.weight", (inter, hidden), init=("uniform", s))
        bb1 = m.tensor(p + "ffn1.bias", (inter,), init=("uniform", s))
        m.layer(Op.LINEAR, [w1, bb1], in0=h, out=f, attr=[Act.GELU_ERF], name=p + "ffn1")
        w2 = m.tensor(p + "ffn2.weight", (hidden, inter), init=("uniform", s))
        bb2 = m.tensor(p + "ffn2.bias", (hidden,), init=("uniform", s))
        m.layer(Op.LINEAR, [w2, bb2], in0=f, in1=h, out=a2, attr=[Act.NONE], name=p + "ffn2")
        g2 = m.tensor(p + "ln2.gamma", (hidden,), init=("range", 0.9, 1.1))
        b2 = m.tensor(p + "ln2.beta", (hidden,), init=("uniform", 0.05))
        m.layer(Op.LAYERNORM, [g2, b2], in0=a2, out=x, attr=[eps12], name=p + "ln2")
    wp = m.tensor("pooler.weight", (hidden, hidden), init=("uniform", s))
    bp = m.tensor("pooler.bias", (hidden,), init=("uniform", s))
    m.layer(Op.LINEAR, [wp, bp], in0=x, out=pooled, attr=[Act.TANH, 0, 1], name="pooler")
    wqa = m.tensor("qa.weight", (2, hidden), init=("uniform", s))
    bqa = m.tensor("qa.bias", (2,), init=("uniform", s))
    m.layer(Op.LINEAR, [wqa, bqa], in0=x, out=logits, attr=[Act.NONE], name="qa")
    m.input_slot, m.output_slot = ids, logits
    return m


def gpt2(n_layers=48, hidden=1600, heads=25, vocab=50257, n_pos=1024, seq=128, seed=4,
         name=None) -> ModelSpec:
    """GPT-2-XL decoder, pre-LN, causal, tied LM head applied to the last token."""
    m = ModelSpec(name or f"gpt2-L{n_layers}-H{hidden}", seed, input_kind=("ids", vocab))
    s = math.sqrt(3.0) * 0.02
    sres = math.sqrt(3.0) * 0.02 / math.sqrt(2 * n_layers)
    inter = 4 * hidden
    ids = m.slot("ids", (seq,), DT_I32)
    x = m.slot("x", (seq, hidden), DT_F32)
    hln = m.slot("ln1_out", (seq, hidden), DT_BF16)
    qkv = m.slot("qkv", (seq, 3 * hidden), DT_BF16)
    ctx = m.slot("ctx", (seq, hidden), DT_BF16)
    a = m.slot("attn_res", (seq, hidden), DT_F32)
    h2 = m.slot("ln2_out", (seq, hidden), DT_BF16)
    f = m.slot("fc_out", (seq, inter), DT_BF16)
    x2 = m.slot("x_next", (seq, hidden), DT_F32)
    xf = m.slot("lnf_out", (seq, hidden), DT_F32)
    logits = m.slot("logits", (1, vocab), DT_F32)
    eps5 = f32_bits(1e-5)

    wte = m.tensor("wte", (vocab, hidden), init=("uniform", s))
    wpe = m.tensor("wpe", (n_pos, hidden), init=("uniform", s))
    m.layer(Op.EMBED, [wte, wpe], in0=ids, out=x, attr=[2, Rule.IDS, Rule.POSITION], name="embed")
    dh = hidden // heads
    cur, nxt = x, x2
    for i in range(n_layers):
        p = f"h{i}."
        g1 = m.tensor(p + "ln_1.gamma", (hidden,), init=("range", 0.9, 1.1))
        b1 = m.tensor(p + "ln_1.beta", (hidden,), init=("uniform", 0.05))
        m.layer(Op.LAYERNORM, [g1, b1], in0=cur, out=hln, attr=[eps5], name=p + "ln_1")
        wa = m.tensor(p + "attn.c_attn.weight", (3 * hidden, hidden), init=("uniform", s))
        ba = m.tensor(p + "attn.c_attn.bias", (3 * hidden,), init=("uniform", s))
        m.layer(Op.LINEAR, [wa, ba], in0=hln, out=qkv, attr=[Act.NONE], name=p + "c_attn")
        m.layer(Op.ATTENTION, [], in0=qkv, out=ctx, attr=[heads, dh, 1], name=p + "attn")
        wp = m.tensor(p + "attn.c_proj.weight", (hidden, hidden), init=("uniform", sres))
        bp = m.tensor(p + "attn.c_proj.bias", (hidden,), init=("uniform", s))
        m.layer(Op.LINEAR, [wp, bp], in0=ctx, in1=cur, out=a, attr=[Act.NONE], name=p + "c_proj")
        g2 = m.tensor(p + "ln_2.gamma", (hidden,), init=("range", 0.9, 1.1))
        b2 = m.tensor(p + "ln_2.beta", (hidden,), init=("uniform", 0.05))
        m.layer(Op.LAYERNORM, [g2, b2], in0=a, out=h2, attr=[eps5], name=p + "ln_2")
        wf = m.tensor(p + "mlp.c_fc.weight", (inter, hidden), init=("uniform", s))
        bf = m.tensor(p + "mlp.c_fc.bias", (inter,), init=("uniform", s))
        m.layer(Op.LINEAR, [wf, bf], in0=h2, out=f, attr=[Act.GELU_TANH], name=p + "c_fc")
        wm = m.tensor(p + "mlp.c_proj.weight", (hidden, inter), init=("uniform", sres))
        bm = m.tensor(p + "mlp.c_proj.bias", (hidden,), init=("uniform", s))
        m.layer(Op.LINEAR, [wm, bm], in0=f, in1=a, out=nxt, attr=[Act.NONE], name=p + "mlp.c_proj")
        cur, nxt = nxt, cur
    gf = m.tensor("ln_f.gamma", (hidden,), init=("range", 0.9, 1.1))
    bfn = m.tensor("ln_f.beta", (hidden,), init=("uniform", 0.05))
    m.layer(Op.LAYERNORM, [gf, bfn], in0=cur, out=xf, attr=[eps5], name="ln_f")
    m.layer(Op.LINEAR, [wte], in0=xf, out=logits, attr=[Act.NONE, seq - 1, 1], name="lm_head")
    m.input_slot, m.output_slot = ids, logits
    return m


def _resnet(stage_blocks, widths, img, stem=64, n_classes=1000, seed=3, name="resnet50") -> ModelSpec:
    """torchvision ResNet v1.5 (stride on the 3x3), BatchNorm folded into conv weight+bias (reading #5)."""
    m = ModelSpec(name, seed, input_kind=("uniform_bf16", 1.0))
    H = img
    x = m.slot("image", (H, H, 3), DT_BF16)

    def he(fan_in, scale=1.0):
        return scale * math.sqrt(3.0) * math.sqrt(2.0 / fan_in)

    def conv(name, src, cin, cout, k, stride, pad, act, res=-1, scale=1.0):
        nonlocal H
        hin = m.slots[src].shape[0]
        hout = (hin + 2 * pad - k) // stride + 1
        w = m.tensor(name + ".weight", (cout, k, k, cin), init=("uniform", he(k * k * cin, scale)))
        b = m.tensor(name + ".bias", (cout,), init=("uniform", 0.05))
        out = m.slot(name + ".out", (hout, hout, cout), DT_BF16)
        m.layer(Op.CONV2D, [w, b], in0=src, in1=res, out=out, attr=[act, stride, pad], name=name)
        return out

    cur = conv("conv1", x, 3, stem, 7, 2, 3, Act.RELU)
    hp = (m.slots[cur].shape[0] + 2 - 3) // 2 + 1
    pooled = m.slot("maxpool.out", (hp, hp, stem), DT_BF16)
    m.layer(Op.MAXPOOL, [], in0=cur, out=pooled, attr=[3, 2, 1], name="maxpool")
    cur, cin = pooled, stem
    for si, (nb, w) in enumerate(zip(stage_blocks, widths)):
        for bi in range(nb):
            stride = 2 if (bi == 0 and si > 0) else 1
            p = f"layer{si + 1}.{bi}"
            c1 = conv(p + ".conv1", cur, cin, w, 1, 1, 0, Act.RELU)
            c2 = conv(p + ".conv2", c1, w, w, 3, stride, 1, Act.RELU)
            if bi == 0:
                sc = conv(p + ".downsample", cur, cin, 4 * w, 1, stride, 0, Act.NONE)
            else:
                sc = cur
            cur = conv(p + ".conv3", c2, w, 4 * w, 1, 1, 0, Act.RELU, res=sc, scale=0.2)
            cin = 4 * w
    feat = m.slot("avgpool.out", (1, cin), DT_F32)
    m.layer(Op.AVGPOOL, [], in0=cur, out=feat, name="avgpool")
    fw = m.tensor("fc.weight", (n_classes, cin), init=("uniform", math.sqrt(3.0) * math.sqrt(1.0 / cin)))
    fb = m.tensor("fc.bias", (n_classes,), init=("uniform", 0.05))
    logits = m.slot("logits", (1, n_classes), DT_F32)
    m.layer(Op.LINEAR, [fw, fb], in0=feat, out=logits, attr=[Act.NONE], name="fc")
    m.input_slot, m.output_slot = x, logits
    return m


def resnet50(seed=3) -> ModelSpec:
    return _resnet([3, 4, 6, 3], [64, 128, 256, 512], 224, seed=seed, name="resnet50")


def resnet101(seed=5) -> ModelSpec:
    """ResNet-101 v1.5 (tab:eval_remote_swap)."""
    return _resnet([3, 4, 23, 3], [64, 128, 256, 512], 224, seed=seed, name="resnet101")


def resnet152(seed=6) -> ModelSpec:
    """ResNet-152 v1.5."""
    return _resnet([3, 8, 36, 3], [64, 128, 256, 512], 224, seed=seed, name="resnet152")


def resnet_tiny(seed=13, img=32) -> ModelSpec:
    """A small ResNet with the same structure (all op kinds, projections, strides) for fast parity."""
    return _resnet([1, 2, 1, 1], [16, 32, 64, 64], img, stem=16, n_classes=40, seed=seed, name=f"resnet_tiny{img}")


def build_model(name: str, seed: Optional[int] = None) -> ModelSpec:
    """A synthetic model of the named configuration; `seed` gives a distinct instance (weights and
    input) of the same architecture, e.g. one per serverless function of a trace."""
    spec = CONFIGS[name]()
    if seed is not None:
        spec.seed = seed
    return spec


CONFIGS: Dict[str, Callable[[], ModelSpec]] = {
    "mlp": lambda: mlp(),
    "bert-base": lambda: bert(),
    "resnet50": lambda: resnet50(),
    "gpt2-xl": lambda: gpt2(),
    # the paper's other swap-evaluation models (tab:eval_remote_swap)
    "resnet101": lambda: resnet101(),
    "resnet152": lambda: resnet152(),
    "bert-large": lambda: bert(n_layers=24, hidden=1024, heads=16, inter=4096, seed=7, name="bert-large"),
    # small members of the same families (parity tests at oracle-friendly sizes)
    "mlp-small": lambda: mlp(width=256, n_layers=3, seed=11),
    "bert-tiny": lambda: bert(n_layers=2, hidden=128, heads=2, inter=256, vocab=1000, max_pos=64, seq=64,
                              seed=12, name="bert-tiny"),
    "gpt2-tiny": lambda: gpt2(n_layers=2, hidden=128, heads=2, vocab=1000, n_pos=64, seq=64, seed=14,
                              name="gpt2-tiny"),
    "gpt2-2L": lambda: gpt2(n_layers=2, seed=15, name="gpt2-xl-2L"),
    "resnet-tiny": lambda: resnet_tiny(),
}
