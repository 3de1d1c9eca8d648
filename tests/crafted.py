"""Crafted exponent patterns shared by the CPU and GPU link-code tests (no method arithmetic)."""
import numpy as np


def tier_offsets(rng, o, n_exc):
    """512 exponent offsets d = h − e whose cheapest code is two-tier with tier-1 offset o: most words in
    [o, o + 3), 80 escapes in [o + 3, 10] and 30 below o, n_exc exceptions (d >= 20), d = 0 at least once."""
    d = rng.integers(o, o + 3, 512)
    idx = rng.permutation(512)
    d[idx[:80]] = rng.integers(o + 3, 11, 80)
    if o:
        d[idx[80:110]] = rng.integers(0, o, 30)
    d[idx[110:110 + n_exc]] = rng.integers(20, 40, n_exc)
    d[idx[511]] = 0  # the block's largest exponent h
    return d


def random_block_mixture(spec, w, seed):
    """Overwrite every 512-word block of every tensor with a block drawn from a random mixture: geometric
    exponent offsets with random ratio and base, two-tier patterns, a narrow band with tiny-value outliers,
    zeros (sprinkled, or the whole block), exponents up to inf / NaN, random 16-bit words."""
    rng = np.random.default_rng(seed)
    for t in spec.tensors:
        words = w[t.offset:t.offset + t.nbytes].view(np.uint16)
        for k in range(0, words.size - 511, 512):
            sm = rng.integers(0, 256, 512).astype(np.uint16)
            kind = rng.integers(0, 6)
            if kind == 0:    # geometric offsets below a random base exponent
                d = np.minimum(rng.geometric(rng.uniform(0.2, 0.8), 512) - 1, 40)
                e = rng.integers(40, 250) - d
            elif kind == 1:  # two-tier friendly
                e = 200 - tier_offsets(rng, int(rng.integers(0, 4)), int(rng.integers(0, 64)))
            elif kind == 2:  # narrow band plus tiny outliers (exceptions)
                e = rng.integers(100, 100 + rng.integers(1, 17), 512)
                e[rng.choice(512, int(rng.integers(0, 100)), replace=False)] = rng.integers(0, 60)
            elif kind == 3:  # zeros sprinkled into a coded block, or an all-zero block
                e = rng.integers(120, 124, 512)
                if rng.random() < 0.3:
                    words[k:k + 512] = 0
                    continue
            elif kind == 4:  # exponents up to inf / NaN
                e = rng.integers(250, 256, 512)
            else:            # random words
                words[k:k + 512] = rng.integers(0, 1 << 16, 512)
                continue
            blk = ((sm & 0x80) << 8) | (np.clip(e, 0, 255).astype(np.uint16) << 7) | (sm & 0x7F)
            if kind == 3:
                blk[rng.random(512) < 0.1] = 0
            words[k:k + 512] = blk
    return w
