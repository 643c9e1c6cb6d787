"""Rows a8-a10: the Monte-Carlo BEM estimator (BEM-MC) — oracle, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md §4.1.1-4.2 step by step (Eq. BIE l.194-198, Eq. SYS l.200-204, the
disk results l.215-236), with the readings of DESIGN.md §3:

a8  Samples, uniform by area (1/q = |Gamma|, l.199).  For sample j (reading R-mc-sample):
      (o0,o1,o2,o3) = Philox4x32-10(ctr = (j, 0, stream_lo, stream_hi), key = seed)
      u_a = (o_a + 0.5) 2^-32
      t   = first index with cdf_t > u0 * cdf_{N-1}          (upper_bound)
      s   = sqrt(u1);  b = (1 - s, s (1 - u2), s u2)
      y_j = (b1 v1 + b2 v2) + b3 v3   (per coordinate, every op rounded)
      n_j = n_t;  g_{m,j} = g_{m,t}  (piecewise-constant Neumann, l.164)
a9/a10  Eq. SYS evaluated at the samples with the disk split (l.215-236), sign of Eq. BM
    with outward normals (reading R-sign):
      eps = sqrt(|Gamma| / (pi M)) unless given          (reading R-eps)
      w   = (|Gamma| - pi eps^2) / (M - 1)               (l.217 "reduction in the
                                                           sampling surface"; R-weight)
      A_ii = 1/2,  A_ij = -w dG/dn_y(y_i, y_j)  (normal at y_j)       (disk dG term = 0, l.236)
      b_i  = -w sum_{j != i} G(y_i, y_j) g_j - (eps/2) g_i            (disk G term, l.231)
    coincident samples (|y_i - y_j| < 1e-12, i != j) raise.
Solve: gmres.gmres.
Parity of the sample *realisation* against truth is statistical only (pinned by the
pulsating-sphere statistics in tests/test_oracle_mc.py); the system and the sampler are
pinned by Philox KATs, on-triangle and per-triangle-frequency checks, M = 1 and g = 0.
"""
import math

import numpy as np

from . import gmres as _gmres
from . import kernel, philox


def sample_uniform(v, t, geom, M, seed, stream_id=0, tag=0):
    """Returns (y (M,3), n (M,3), tri (M,) int32).  tag 0: boundary samples (a8); tag 2:
    Poisson-disk candidates (oracle/poisson.py)."""
    v = np.asarray(v, dtype=np.float64)
    t = np.asarray(t, dtype=np.int64)
    u = philox.uniforms(np.arange(M), tag, stream_id, seed)
    cdf = geom["cdf"]
    tri = np.searchsorted(cdf, u[:, 0] * cdf[-1], side="right")
    tri = np.minimum(tri, len(cdf) - 1)
    s = np.sqrt(u[:, 1])
    b1 = 1.0 - s
    b2 = s * (1.0 - u[:, 2])
    b3 = s * u[:, 2]
    v1, v2, v3 = v[t[tri, 0]], v[t[tri, 1]], v[t[tri, 2]]
    y = (b1[:, None] * v1 + b2[:, None] * v2) + b3[:, None] * v3
    return y, geom["normal"][tri].copy(), tri.astype(np.int32)


def default_eps(total_area, M):
    return math.sqrt(total_area / (math.pi * M))


def weight(total_area, M, eps):
    return (total_area - math.pi * eps * eps) / (M - 1) if M > 1 else 0.0


def check_coincident(y):
    M = y.shape[0]
    for i in range(M):
        d = np.sqrt(np.sum((y - y[i]) ** 2, axis=1))
        d[i] = np.inf
        j = int(np.argmin(d))
        if d[j] < kernel.SINGULAR_R:
            raise ZeroDivisionError(f"coincident samples ({i}, {j})")


def system(y, n, g, k, total_area, eps=None):
    """Dense Eq. SYS: returns (A (M,M), b (M,)) for one wavenumber k, Neumann g (M,)."""
    M = y.shape[0]
    eps = default_eps(total_area, M) if eps is None or eps <= 0 else eps
    w = weight(total_area, M, eps)
    check_coincident(y)
    A = np.zeros((M, M), np.complex128)
    b = np.zeros(M, np.complex128)
    g = np.asarray(g, dtype=np.complex128)
    for i in range(M):
        j = np.arange(M) != i
        A[i, j] = -w * kernel.green_dn_y(y[i], y[j], n[j], k)
        A[i, i] = 0.5
        b[i] = -w * np.sum(kernel.green(y[i], y[j], k) * g[j]) - 0.5 * eps * g[i]
    return A, b


def surface_pressure(v, t, geom, ks, g_tri, M, seed, stream_id=0, eps=None,
                     tol=1e-6, max_iter=200, samples=None):
    """nat_mc_surface_pressure: returns (y, n, tri, p (n_sys, M), infos)."""
    if samples is None:
        y, n, tri = sample_uniform(v, t, geom, M, seed, stream_id)
    else:
        y, n, tri = samples
    g_tri = np.atleast_2d(np.asarray(g_tri, dtype=np.complex128))
    p = np.zeros((len(ks), y.shape[0]), np.complex128)
    infos = []
    for m, k in enumerate(ks):
        g = g_tri[m][tri]
        A, b = system(y, n, g, k, geom["total_area"], eps)
        x, info = _gmres.gmres(lambda z: A @ z, b, tol, max_iter)
        p[m] = x
        infos.append(info)
    return y, n, tri, p, infos
