"""oracle/philox.py -- TEST INFRASTRUCTURE ONLY.

Philox4x32-10 counter-based generator (Salmon, Moraes, Dror, Shaw, "Parallel random
numbers: as easy as 1, 2, 3", SC'11), written here from its published definition and
independently of the CUDA product path, which implements the same generator in
paper_2308_15020_b200/csrc.  Both sides draw the random phase of PAPER.md's rephasing
heuristic ("a point randomly sampled from [-1,1]^n") and the initial sample of
Alg. 1 line 1 from this generator, keyed as DESIGN.md "RNG" states:

    key     = (seed & 0xffffffff, seed >> 32)
    counter = (i // 4, global point index, round, 0x51A7)   # word i % 4 of the output
    value   = ((word >> 8) + 0.5) * 2^-23 - 1               # in (-1, 1), exact in fp32
"""
from __future__ import annotations

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF
STREAM_TAG = 0x51A7


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = (int(v) & MASK for v in ctr)
    k0, k1 = (int(v) & MASK for v in key)
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK
        hi1, lo1 = p1 >> 32, p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK, lo1, (hi0 ^ c3 ^ k1) & MASK, lo0
    return c0, c1, c2, c3


def uniform_pm1(seed: int, point: int, rnd: int, n: int):
    """n values in (-1, 1) for (seed, global point, round)."""
    key = (seed & MASK, (seed >> 32) & MASK)
    out = []
    for blk in range((n + 3) // 4):
        words = philox4x32_10((blk, point, rnd, STREAM_TAG), key)
        for w in words:
            if len(out) < n:
                out.append(((w >> 8) + 0.5) * 2.0 ** -23 - 1.0)
    return out
