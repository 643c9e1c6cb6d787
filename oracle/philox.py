"""Philox4x32-10 counter-based generator (oracle, NumPy uint64 arithmetic).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3", SC'11:
  multipliers M0 = 0xD2511F53, M1 = 0xCD9E8D57; Weyl increments W0 = 0x9E3779B9,
  W1 = 0xBB67AE85; round (c0,c1,c2,c3) <- (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2),
  hi(M0 c0) ^ c3 ^ k1, lo(M0 c0)); the key is bumped between rounds; 10 rounds.
The MC sampler draws its uniforms from this stream (DESIGN.md §3 reading R-mc-sample,
PAPER.md l.199 "uniform sampling"), so CPU and GPU draw identical samples.
Pinned by the Random123 known-answer tests in tests/test_oracle_philox.py.
"""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
SH = np.uint64(32)


def philox4x32_10(ctr, key):
    """ctr: (...,4) integer array, key: (2,) ints.  Returns (...,4) uint32 as uint64."""
    c = [np.asarray(ctr, dtype=np.uint64)[..., i] & MASK for i in range(4)]
    k0 = np.uint64(int(key[0]) & 0xFFFFFFFF)
    k1 = np.uint64(int(key[1]) & 0xFFFFFFFF)
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [((p1 >> SH) ^ c[1] ^ k0) & MASK, p1 & MASK,
             ((p0 >> SH) ^ c[3] ^ k1) & MASK, p0 & MASK]
    return np.stack(c, axis=-1)


def uniforms(index, tag, stream_id, seed):
    """u_a = (o_a + 0.5) 2^-32, exact in fp64, for counter (index, tag, stream_lo,
    stream_hi) and key (seed_lo, seed_hi).  index: int array.  Returns (...,4) float64."""
    index = np.asarray(index, dtype=np.uint64)
    ctr = np.zeros(index.shape + (4,), dtype=np.uint64)
    ctr[..., 0] = index & MASK
    ctr[..., 1] = np.uint64(tag)
    ctr[..., 2] = np.uint64(int(stream_id) & 0xFFFFFFFF)
    ctr[..., 3] = np.uint64((int(stream_id) >> 32) & 0xFFFFFFFF)
    o = philox4x32_10(ctr, (int(seed) & 0xFFFFFFFF, (int(seed) >> 32) & 0xFFFFFFFF))
    return (o.astype(np.float64) + 0.5) * 2.0 ** -32
