"""Rows a4 + a5 (dense collocation BEM assembly) and a6 (matvec) — oracle, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Equation: the conventional BIE, i.e. Eq. BM with beta = 0
("i.e., beta = 0", l.191), with outward normals (reading R-sign):
    1/2 p(x) - int_Gamma p(y) dG/dn_y(x,y) dS(y) = - int_Gamma dp/dn(y) G(x,y) dS(y).
Discretisation (reading R-colloc; the paper's bempp/Galerkin details are
not given): piecewise-constant p_t, g_t; collocation at the centroids c_i:
    A p = b,   A_ij = 1/2 delta_ij - K_ij,   b_i = - sum_j V_ij g_j,
    K_ij = int_{T_j} dG/dn_y(c_i, y) dS,   V_ij = int_{T_j} G(c_i, y) dS.
Quadrature by pair class ("adjacent or identical elements"):
    far      : rule ``far_pts`` (default R3) on T_j
    class N  : ``near_levels_N`` (default 1) midpoint subdivisions x R7
    class S  : ``near_levels_S`` (default 3) midpoint subdivisions x R7
    self     : K_ii = 0, V_ii by the polar rule of quadrature.self_single_layer
The oracle forms every entry directly with its final rule (no far-then-correct).
Pinned by tests/test_oracle_bem.py: Gauss identity at k = 0, sphere eigenvalues of V
and K, brute-force entries on tiny meshes, pulsating/oscillating sphere and interior
point-source solutions within 2%.
"""
import numpy as np

from . import kernel, nearlist, quadrature

DEFAULTS = dict(far_pts=3, near_levels_S=3, near_levels_N=1, near_eta=4.0, self_theta_pts=16)


def _opts(opts):
    o = dict(DEFAULTS)
    if opts:
        o.update({k: v for k, v in opts.items() if v})
    return o


def _entries(x, v1, v2, v3, n, area, lam, w, k):
    """K, V for one collocation point x against triangles (m,3) with rule (lam, w)."""
    # points (m, Q, 3)
    y = (lam[None, :, 0:1] * v1[:, None, :] + lam[None, :, 1:2] * v2[:, None, :]) \
        + lam[None, :, 2:3] * v3[:, None, :]
    G = kernel.green(x[None, None, :], y, k)
    dG = kernel.green_dn_y(x[None, None, :], y, n[:, None, :], k)
    K = area * np.sum(w[None, :] * dG, axis=1)
    V = area * np.sum(w[None, :] * G, axis=1)
    return K, V


def assemble(v, t, geom, k, g=None, rows=None, opts=None, near=None, return_V=False):
    """Rows ``rows`` (default all) of A and b = -V g.

    v (V,3), t (N,3); geom from geometry.mesh_prepare; g (n_rhs, N) complex or None.
    Returns A (len(rows), N) complex128, b (n_rhs, len(rows)) [, V rows]."""
    o = _opts(opts)
    v = np.asarray(v, dtype=np.float64)
    t = np.asarray(t, dtype=np.int64)
    N = t.shape[0]
    rows = np.arange(N) if rows is None else np.asarray(rows)
    V1, V2, V3 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    c, nrm, area = geom["centroid"], geom["normal"], geom["area"]
    lam_f, w_f = quadrature.rule(o["far_pts"])
    lam_s, w_s = quadrature.composite_rule(o["near_levels_S"], 7)
    lam_n, w_n = quadrature.composite_rule(o["near_levels_N"], 7)
    if near is None:
        near = nearlist.near_list(t, c, geom["diam"], o["near_eta"], rows=rows)
    rp, col, cls = near
    A = np.zeros((len(rows), N), dtype=np.complex128)
    Vm = np.zeros((len(rows), N), dtype=np.complex128)
    for r, i in enumerate(rows):
        x = c[i]
        idx = np.arange(N)
        idx = idx[idx != i]
        K, V = np.zeros(N, np.complex128), np.zeros(N, np.complex128)
        K[idx], V[idx] = _entries(x, V1[idx], V2[idx], V3[idx], nrm[idx], area[idx],
                                  lam_f, w_f, k)
        js, cl = col[rp[r]:rp[r + 1]], cls[rp[r]:rp[r + 1]]
        for code, lam, w in ((nearlist.CLS_S, lam_s, w_s), (nearlist.CLS_N, lam_n, w_n)):
            j = js[cl == code]
            if j.size:
                K[j], V[j] = _entries(x, V1[j], V2[j], V3[j], nrm[j], area[j], lam, w, k)
        K[i] = 0.0
        V[i] = quadrature.self_single_layer(V1[i], V2[i], V3[i], k, o["self_theta_pts"])
        A[r] = -K
        A[r, i] += 0.5
        Vm[r] = V
    b = None
    if g is not None:
        g = np.atleast_2d(np.asarray(g, dtype=np.complex128))
        b = -(Vm @ g.T).T
    return (A, b, Vm) if return_V else (A, b)


def matvec(A, x):
    """Row a6: y = A x (plain definition)."""
    return np.asarray(A) @ np.asarray(x)
