"""Row a1: mesh preparation (oracle, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper builds "the scene ... surface triangle mesh" with per-triangle Neumann data
(PAPER.md l.164); the per-triangle quantities below are the standard flat-triangle ones
(DESIGN.md §3 reading R-geom).  Arithmetic order is fixed (no fused multiply-add: NumPy
rounds every operation) so that the integer decisions that depend on these values
(near list, sample -> triangle) are reproducible bit for bit:

  e   = (v2 - v1) x (v3 - v1), each component (a_y*b_z) - (a_z*b_y)
  |e| = sqrt((e_x*e_x + e_y*e_y) + e_z*e_z),  area = 0.5*|e|,  n = e / |e|
  c   = ((v1 + v2) + v3) / 3
  diam = longest edge, each length sqrt((d_x*d_x + d_y*d_y) + d_z*d_z)
  cdf  = sequential prefix sum of area (np.cumsum),  |Gamma| = cdf[-1]
  centre = sum_t A_t c_t / |Gamma|, each sum sequential left to right over t (the
           definition's order, as for the cdf; np.cumsum is that sequential accumulate),
  R = max_vertices sqrt((dx*dx + dy*dy) + dz*dz),  d = v - centre
Validation: every area > 0; signed volume sum_t v1.(v2 x v3)/6 > 0 (outward).
Pinned by tests/test_oracle_geometry.py (sphere area/volume convergence, hand triangle,
closed-surface identity sum A n = 0).
"""
import numpy as np


def _cross(a, b):
    return np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
                     a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                     a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)


def _norm(d):
    return np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])


def mesh_prepare(v, t):
    """v: (V,3) float64, t: (N,3) int.  Returns dict of per-triangle arrays + scalars."""
    v = np.asarray(v, dtype=np.float64)
    t = np.asarray(t, dtype=np.int64)
    v1, v2, v3 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    e = _cross(v2 - v1, v3 - v1)
    en = _norm(e)
    if np.any(~(en > 0)):
        bad = int(np.flatnonzero(~(en > 0))[0])
        raise ValueError(f"zero-area triangle {bad}")
    area = 0.5 * en
    normal = e / en[:, None]
    centroid = ((v1 + v2) + v3) / 3.0
    diam = np.maximum(np.maximum(_norm(v2 - v1), _norm(v3 - v2)), _norm(v1 - v3))
    vol = np.sum(np.sum(v1 * _cross(v2, v3), axis=1)) / 6.0
    if not vol > 0:
        raise ValueError("mesh is not outward-oriented (signed volume <= 0)")
    cdf = np.cumsum(area)
    total = float(cdf[-1])
    ac = area[:, None] * centroid
    centre = np.array([np.cumsum(ac[:, d])[-1] for d in range(3)]) / total
    dv = v - centre[None, :]
    R = float(np.max(_norm(dv)))
    return dict(centroid=centroid, normal=normal, area=area, diam=diam, cdf=cdf,
                total_area=total, center=centre, bound_radius=R, volume=float(vol))
