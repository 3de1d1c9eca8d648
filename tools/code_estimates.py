"""Coded size of a model's store under candidate exponent codes, from the block histograms alone
(numpy; no libfsw): format v3 (frame of reference), v4 (+ two-tier), a per-level unary code, and the
empirical-entropy floor (8 bits of sign|mantissa + the entropy of each block's exponent histogram).

    python tools/code_estimates.py [bert-base resnet50 ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def pad16(x):
    return (x + 15) // 16 * 16


def estimates(words):
    blk = words[: words.size // 512 * 512].reshape(-1, 512)
    e = ((blk >> 7) & 0xFF).astype(np.int32)
    d = e.max(1, keepdims=True) - e
    zero = (blk == 0).all(1)
    v3 = np.full(len(blk), 1024)
    for b in range(5):
        v3 = np.minimum(v3, 512 + pad16(64 * b + 4 * (d >= (1 << b)).sum(1)))
    v4 = v3.copy()
    nx = (d >= 11).sum(1)
    for o in range(4):
        ne = ((d < o) | (d >= o + 3)).sum(1)
        v4 = np.minimum(v4, np.where(nx <= 63, 512 + pad16(128 + 12 * ((ne + 31) // 32) + 4 * nx), 4096))
    un = v4.copy()
    for order in ([1, 2, 0, 3, 4, 5, 6, 7], [0, 1, 2, 3, 4, 5, 6, 7], [2, 3, 1, 4, 0, 5, 6, 7]):
        rank = np.full(256, 99)
        rank[order] = np.arange(len(order))
        r = rank[np.minimum(d, 255)]
        L = len(order)
        tot = sum(4 * (((r >= k).sum(1) + 31) // 32) for k in range(L))
        x = (r >= L).sum(1)
        un = np.minimum(un, np.where(x <= 63, 512 + pad16(tot + 4 * x), 4096))
    sample = blk[np.random.default_rng(0).choice(len(blk), min(4000, len(blk)), replace=False)]
    bits = 0.0
    for row in sample:
        if row.any():
            c = np.bincount((row >> 7) & 0xFF)
            p = c[c > 0] / 512.0
            bits += 8.0 - (p * np.log2(p)).sum()
    raw = blk.size * 2
    f = lambda v: float(np.where(zero, 0, v).sum() / raw)
    # one static frequency table over d (clamped to 15) for the whole store: the ideal cost of an entropy coder
    # (e.g. interleaved rANS) that ships one table per tensor / layer instead of adapting per block
    dc = np.minimum(d, 15)
    c = np.bincount(dc.ravel(), minlength=16).astype(np.float64) + 0.5
    q = c / c.sum()
    static = float((blk.shape[0] * 512 * 8 + (-np.log2(q[dc])).sum()) / (raw * 8))
    return f(v3), f(v4), f(un), bits / len(sample) / 16.0, static


for name in sys.argv[1:] or ["bert-base", "resnet50"]:
    spec = synth.build_model(name)
    w = spec.build_weights()
    v3, v4, un, floor, static = estimates(np.frombuffer(np.asarray(w).tobytes(), dtype=np.uint16))
    print(f"{name:10s} v3 {v3:.4f}  v4 {v4:.4f}  unary(8 levels) {un:.4f}  one static table {static:.4f}  "
          f"per-block entropy floor {floor:.4f}", flush=True)
