"""NEXT-3: Poisson-disk boundary samples (oracle, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md l.214: "we use parallel Poisson disk sampling [bowers2010], ensuring more uniform
sample distribution"; l.402: Poisson sampling costs ~10 ms against ~1 ms for random
sampling and converges faster.  The paper gives no radius or candidate rule; reading
R-poisson follows SPEC's design decisions (r = 0.7 sqrt(|Gamma| / M_target),
30 darts per requested sample) and Bowers et al.'s phase-group parallelisation, which makes
the result independent of the processing order:

1. Candidates c = 0 .. 30 M_target - 1: the a8 construction with Philox tag 2
   (counter (c, 2, stream_lo, stream_hi), key = seed): triangle by the area CDF, uniform
   barycentric point, the triangle's normal.
2. Grid: cell size h = r / sqrt(3) over the cube centre +- R (R = bounding radius),
   i_d = min(floor((x_d - (centre_d - R)) / h), n - 1), n = floor(2R / h) + 1 per axis.  A
   cell's diagonal is r, so it holds at most one accepted sample; two cells whose indices
   differ by >= 3 along an axis are >= 2h > r apart, so conflicts only occur inside the
   5 x 5 x 5 neighbourhood, and cells in the same phase (i_x mod 3, i_y mod 3, i_z mod 3)
   never conflict with each other.
3. Each cell lists its candidates by ascending index.  For trial t = 0, 1, ... and phase
   p = (i_x mod 3) + 3 (i_y mod 3) + 9 (i_z mod 3) = 0..26: every empty cell of phase p
   with more than t candidates tests its t-th candidate against the accepted samples of
   its 5^3 neighbourhood and accepts it when all squared distances
   ((dx dx + dy dy) + dz dz) (fp64, each op rounded) are >= r^2 (r^2 = r r).
   Cells of one phase are independent, so the loop over them may run in any order
   (`order` below shuffles it: the result must not change).
4. The accepted candidates, ascending by candidate index, are the samples (M of them).

Pinned by tests/test_oracle_poisson.py: minimum distance >= r by brute force, maximality
over the candidate pool (every candidate lies within r of a sample), points on their
triangles, count vs M_target, invariance under the in-phase processing order.
"""
import math

import numpy as np

from . import mc

N_CAND_PER_TARGET = 30


def default_radius(total_area, M_target):
    return 0.7 * math.sqrt(total_area / M_target)


def grid_of(centre, R, r):
    h = r / math.sqrt(3.0)
    n = int(math.floor(2.0 * R / h)) + 1
    origin = np.asarray(centre, dtype=np.float64) - R
    return h, n, origin


def cell_index(y, origin, h, n):
    q = np.floor((y - origin[None, :]) / h).astype(np.int64)
    return np.clip(q, 0, n - 1)


def sample(v, t, geom, M_target, seed, stream_id=0, r=None, order=None):
    """Returns (y (M,3), n (M,3), tri (M,), cand (M,) candidate indices, r).
    order: optional np.random.Generator shuffling the in-phase cell order (test only)."""
    r = default_radius(geom["total_area"], M_target) if r is None or r <= 0 else float(r)
    n_cand = N_CAND_PER_TARGET * M_target
    y, nrm, tri = mc.sample_uniform(v, t, geom, n_cand, seed, stream_id, tag=2)
    centre, R = geom["center"], geom["bound_radius"]
    h, n, origin = grid_of(centre, R, r)
    ijk = cell_index(y, origin, h, n)
    key = (ijk[:, 2] * n + ijk[:, 1]) * n + ijk[:, 0]
    perm = np.argsort(key, kind="stable")              # candidates by cell, then by index
    keys, start, cnt = np.unique(key[perm], return_index=True, return_counts=True)
    cells = np.stack([keys % n, (keys // n) % n, keys // (n * n)], axis=1)
    phase = (cells[:, 0] % 3) + 3 * (cells[:, 1] % 3) + 9 * (cells[:, 2] % 3)
    acc = np.full(len(keys), -1, dtype=np.int64)      # accepted candidate per cell
    slot = {int(k): i for i, k in enumerate(keys)}
    r2 = r * r
    offs = [(dx, dy, dz) for dz in range(-2, 3) for dy in range(-2, 3) for dx in range(-2, 3)]
    for tr in range(int(cnt.max())):
        for p in range(27):
            idx = np.nonzero((phase == p) & (acc < 0) & (cnt > tr))[0]
            if order is not None:
                idx = order.permutation(idx)
            for ci in idx:
                c = perm[start[ci] + tr]
                x, yy, z = cells[ci]
                ok = True
                for dx, dy, dz in offs:
                    a, b, e = x + dx, yy + dy, z + dz
                    if not (0 <= a < n and 0 <= b < n and 0 <= e < n):
                        continue
                    nb = slot.get(int((e * n + b) * n + a))
                    if nb is None or acc[nb] < 0:
                        continue
                    d = y[c] - y[acc[nb]]
                    if (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2] < r2:
                        ok = False
                        break
                if ok:
                    acc[ci] = c
    cand = np.sort(acc[acc >= 0])
    return y[cand], nrm[cand], tri[cand], cand, r
