"""Row a2: near list by brute force (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's CUDA BEM treats "integrations involving adjacent or identical elements"
separately.  Reading R-near: for row i, source triangle
j != i is
  class S (=1) if T_j shares >= 1 vertex index with T_i (welded meshes; integer test),
  class N (=2) otherwise, if |c_i - c_j| < eta * diam_j  (strict <, fp64, no FMA:
              sqrt((dx*dx + dy*dy) + dz*dz), dx = c_i.x - c_j.x),
  far        otherwise (not listed).
CSR, columns ascending within each row.  O(N^2) distance tests.
Pinned by tests/test_oracle_nearlist.py (vertex-valence count of class S on the
icosphere; every listed N pair meets the predicate and no unlisted pair does, checked
with an independent KD-tree query).
"""
import numpy as np

CLS_S, CLS_N = 1, 2


def near_list(t, centroid, diam, eta=4.0, rows=None):
    t = np.asarray(t, dtype=np.int64)
    n = t.shape[0]
    rows = range(n) if rows is None else rows
    row_ptr, cols, cls = [0], [], []
    thr = eta * diam
    for i in rows:
        shares = np.zeros(n, dtype=bool)
        for a in range(3):
            shares |= np.any(t == t[i, a], axis=1)
        shares[i] = False
        d = centroid[i][None, :] - centroid
        dist = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
        near = (dist < thr) & ~shares
        near[i] = False
        j = np.flatnonzero(shares | near)
        cols.append(j)
        cls.append(np.where(shares[j], CLS_S, CLS_N))
        row_ptr.append(row_ptr[-1] + j.size)
    return (np.array(row_ptr, dtype=np.int64),
            np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32),
            np.concatenate(cls).astype(np.uint8) if cls else np.zeros(0, np.uint8))
