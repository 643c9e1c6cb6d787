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

NEXT-1, Burton-Miller (``bm=True``): Eq. BM exactly as printed (l.176-177), beta = i/k,
with outward normals (reading R-bm):
    1/2 p - K p - beta W p = -V g - beta K' g - (beta/2) g,
    K'_ij = int_{T_j} dG/dn_x(c_i, y) dS,  W_ij = int_{T_j} d2G/dn_x dn_y(c_i, y) dS,
same rules per class; self: K'_ii = 0 (flat triangle), W_ii by the polar finite part of
quadrature.self_hypersingular.  Pinned by tests/test_oracle_bm.py (finite-difference
kernels, the finite part against a punctured polar integral, sphere eigenvalues of W and
K', solutions at a CBIE-singular wavenumber).
"""
import numpy as np

from . import kernel, nearlist, quadrature

DEFAULTS = dict(far_pts=3, near_levels_S=3, near_levels_N=1, near_eta=4.0, self_theta_pts=16)


def _opts(opts):
    o = dict(DEFAULTS)
    if opts:
        o.update({k: v for k, v in opts.items() if v})
    return o


def _entries(x, v1, v2, v3, n, area, lam, w, k, nx=None):
    """K, V (and with the collocation normal nx also K', W) for one collocation point x
    against triangles (m,3) with rule (lam, w)."""
    # points (m, Q, 3)
    y = (lam[None, :, 0:1] * v1[:, None, :] + lam[None, :, 1:2] * v2[:, None, :]) \
        + lam[None, :, 2:3] * v3[:, None, :]
    G = kernel.green(x[None, None, :], y, k)
    dG = kernel.green_dn_y(x[None, None, :], y, n[:, None, :], k)
    K = area * np.sum(w[None, :] * dG, axis=1)
    V = area * np.sum(w[None, :] * G, axis=1)
    if nx is None:
        return K, V
    dGx = kernel.green_dn_x(x[None, None, :], y, nx[None, None, :], k)
    d2G = kernel.green_dn_x_dn_y(x[None, None, :], y, nx[None, None, :], n[:, None, :], k)
    Kp = area * np.sum(w[None, :] * dGx, axis=1)
    W = area * np.sum(w[None, :] * d2G, axis=1)
    return K, V, Kp, W


def assemble(v, t, geom, k, g=None, rows=None, opts=None, near=None, return_V=False, bm=False):
    """Rows ``rows`` (default all) of A and b = -V g (bm: the Burton-Miller A and b).

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
    if bm and not k > 0:
        raise ValueError("Burton-Miller needs k > 0 (beta = i/k)")
    beta = 1j / k if bm else 0.0
    A = np.zeros((len(rows), N), dtype=np.complex128)
    Vm = np.zeros((len(rows), N), dtype=np.complex128)   # V (+ beta K' with bm): the RHS operator
    for r, i in enumerate(rows):
        x = c[i]
        nx = nrm[i] if bm else None
        idx = np.arange(N)
        idx = idx[idx != i]
        K, V = np.zeros(N, np.complex128), np.zeros(N, np.complex128)
        Kp, W = np.zeros(N, np.complex128), np.zeros(N, np.complex128)
        parts = [(idx, lam_f, w_f)]
        js, cl = col[rp[r]:rp[r + 1]], cls[rp[r]:rp[r + 1]]
        for code, lam, w in ((nearlist.CLS_S, lam_s, w_s), (nearlist.CLS_N, lam_n, w_n)):
            j = js[cl == code]
            if j.size:
                parts.append((j, lam, w))
        for j, lam, w in parts:     # near rules overwrite the far ones
            e = _entries(x, V1[j], V2[j], V3[j], nrm[j], area[j], lam, w, k, nx)
            K[j], V[j] = e[0], e[1]
            if bm:
                Kp[j], W[j] = e[2], e[3]
        K[i] = 0.0
        V[i] = quadrature.self_single_layer(V1[i], V2[i], V3[i], k, o["self_theta_pts"])
        if bm:
            Kp[i] = 0.0
            W[i] = quadrature.self_hypersingular(V1[i], V2[i], V3[i], k, o["self_theta_pts"])
        A[r] = -K - beta * W
        A[r, i] += 0.5
        Vm[r] = V + beta * Kp
    b = None
    if g is not None:
        g = np.atleast_2d(np.asarray(g, dtype=np.complex128))
        b = -(Vm @ g.T).T
        if bm:
            b -= 0.5 * beta * g[:, rows]
    return (A, b, Vm) if return_V else (A, b)


def matvec(A, x):
    """Row a6: y = A x (plain definition)."""
    return np.asarray(A) @ np.asarray(x)
