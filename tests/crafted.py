"""Crafted exponent patterns shared by the CPU and GPU link-code tests (no method arithmetic)."""


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
