"""NEXT-2: Galerkin P0 assembly of the conventional BIE — oracle, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper "reengineer[s] the boundary element method" of bempp:
a Galerkin discretisation whose element-pair integrals run on the GPU, one CUDA block
per element pair for "adjacent or identical elements" (l.187).  The rules are not
given; this module is the build's reading R-galerkin:

Equation (Eq. BM with beta = 0, l.176-177, l.191; outward normals, reading R-sign),
tested with the indicator of each triangle (P0 test = trial space):
    sum_j A_ij p_j = b_i,   A_ij = 1/2 |T_i| delta_ij - K_ij,   b_i = - sum_j V_ij g_j,
    K_ij = int_{T_i} int_{T_j} dG/dn_y(x, y) dS_y dS_x,   V_ij = int_{T_i} int_{T_j} G dS_y dS_x.
Quadrature by pair class (the near list of oracle/nearlist.py, eta = 4):
    far     : tensor product of the ``far_pts`` rule (R3) on T_i and on T_j   (9 points)
    class N : tensor product of ``near_levels_N`` subdivisions x R7 on both   (28 x 28)
    class S : Sauter-Schwab (Sauter & Schwab, Boundary Element Methods, §5.2) with
              ``ss_order`` Gauss-Legendre points per cube dimension: common edge (5
              regions) when the pair shares 2 vertices, common vertex (2 regions) when
              it shares 1
    self    : Sauter-Schwab identical panels (6 regions); K_ii = 0 on a flat triangle
Sauter-Schwab parametrisation: reference triangle tau = {0 <= x2 <= x1 <= 1},
chi(x) = a + x1 (b - a) + x2 (c - b), |det| = 2 |T|; for the shared edge / vertex the
two triangles list the shared vertices first in the same order, so chi_i(s, 0) =
chi_j(s, 0) (edge) or chi_i(0) = chi_j(0) (vertex).
Pinned by tests/test_oracle_galerkin.py: rule weights and separable monomials over
tau x tau for every case, the k = 0 single layer of coplanar identical / edge / vertex
pairs against the closed-form in-plane potential of a triangle integrated over the test
triangle, the Gauss identity sum_j K_ij = -|T_i|/2 at k = 0, brute-force far entries,
and Galerkin solutions of the pulsating / oscillating sphere within 2 % of the analytic
fields.
"""
import functools

import numpy as np

from . import kernel, nearlist, quadrature

DEFAULTS = dict(far_pts=3, near_levels_N=1, near_eta=4.0, ss_order=4)


def _opts(opts):
    o = dict(DEFAULTS)
    if opts:
        o.update({k: v for k, v in opts.items() if v})
    return o


def _gl01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return (x + 1.0) / 2.0, w / 2.0


@functools.lru_cache(maxsize=None)
def ss_rule(case: str, n: int):
    """Sauter-Schwab points on tau x tau: (xh (P,2), yh (P,2), w (P,)); the weights
    include the Jacobians of the cube maps, so sum(w) = |tau|^2 = 1/4."""
    g, wg = _gl01(n)
    xi, e1, e2, e3 = (a.ravel() for a in np.meshgrid(g, g, g, g, indexing="ij"))
    w4 = np.einsum("a,b,c,d->abcd", wg, wg, wg, wg).ravel()
    P = lambda a, b: np.stack([a, b], axis=1)
    regs = []
    if case == "identical":
        f = w4 * xi ** 3 * e1 ** 2 * e2
        regs = [
            (P(xi, xi * (1 - e1 + e1 * e2)), P(xi * (1 - e1 * e2 * e3), xi * (1 - e1)), f),
            (P(xi * (1 - e1 * e2 * e3), xi * (1 - e1)), P(xi, xi * (1 - e1 + e1 * e2)), f),
            (P(xi, xi * e1 * (1 - e2 + e2 * e3)), P(xi * (1 - e1 * e2), xi * e1 * (1 - e2)), f),
            (P(xi * (1 - e1 * e2), xi * e1 * (1 - e2)), P(xi, xi * e1 * (1 - e2 + e2 * e3)), f),
            (P(xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), P(xi, xi * e1 * (1 - e2)), f),
            (P(xi, xi * e1 * (1 - e2)), P(xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), f),
        ]
    elif case == "edge":
        f1 = w4 * xi ** 3 * e1 ** 2
        f = w4 * xi ** 3 * e1 ** 2 * e2
        regs = [
            (P(xi, xi * e1 * e3), P(xi * (1 - e1 * e2), xi * e1 * (1 - e2)), f1),
            (P(xi, xi * e1), P(xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), f),
            (P(xi * (1 - e1 * e2), xi * e1 * (1 - e2)), P(xi, xi * e1 * e2 * e3), f),
            (P(xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), P(xi, xi * e1), f),
            (P(xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), P(xi, xi * e1 * e2), f),
        ]
    elif case == "vertex":
        f = w4 * xi ** 3 * e2
        regs = [
            (P(xi, xi * e1), P(xi * e2, xi * e2 * e3), f),
            (P(xi * e2, xi * e2 * e3), P(xi, xi * e1), f),
        ]
    else:
        raise ValueError(case)
    xh = np.concatenate([r[0] for r in regs])
    yh = np.concatenate([r[1] for r in regs])
    w = np.concatenate([r[2] for r in regs])
    for a in (xh, yh, w):
        a.flags.writeable = False   # cached: shared by every call
    return xh, yh, w


def chi(a, b, c, xh):
    """Sauter-Schwab map of the reference triangle onto (a, b, c): a + x1 (b - a) + x2 (c - b)."""
    return a[None, :] + xh[:, 0:1] * (b - a)[None, :] + xh[:, 1:2] * (c - b)[None, :]


def ordered_pair(ti, tj):
    """Vertex orders of (T_i, T_j) with the shared vertices first, in T_i's order, and the
    Sauter-Schwab case."""
    ti, tj = list(ti), list(tj)
    shared = [a for a in ti if a in tj]
    if len(shared) == 3:
        return ti, ti, "identical"
    oi = shared + [a for a in ti if a not in shared]
    oj = shared + [a for a in tj if a not in shared]
    return oi, oj, {2: "edge", 1: "vertex"}[len(shared)]


def ss_entry(v, ti, tj, n_j, area_i, area_j, k, n):
    """(K_ij, V_ij) of a pair sharing a vertex, an edge or identical, by Sauter-Schwab."""
    oi, oj, case = ordered_pair(ti, tj)
    xh, yh, w = ss_rule(case, n)
    x = chi(v[oi[0]], v[oi[1]], v[oi[2]], xh)
    y = chi(v[oj[0]], v[oj[1]], v[oj[2]], yh)
    jac = (2.0 * area_i) * (2.0 * area_j)
    V = jac * np.sum(w * kernel.green(x, y, k))
    K = jac * np.sum(w * kernel.green_dn_y(x, y, n_j[None, :], k))
    return K, V


def tensor_entries(Xi, wi, area_i, Y, wy, nrm, area_j, k):
    """(K, V) of one test triangle (points Xi (Qi,3), weights wi summing to 1) against
    triangles with points Y (m,Qj,3), weights wy (Qj,), normals (m,3)."""
    G = kernel.green(Xi[None, :, None, :], Y[:, None, :, :], k)
    dG = kernel.green_dn_y(Xi[None, :, None, :], Y[:, None, :, :], nrm[:, None, None, :], k)
    W = wi[:, None] * wy[None, :]
    V = area_i * area_j * np.einsum("ab,mab->m", W, G)
    K = area_i * area_j * np.einsum("ab,mab->m", W, dG)
    return K, V


def assemble(v, t, geom, k, g=None, rows=None, opts=None, near=None):
    """Rows ``rows`` (default all) of the Galerkin A and b = -V g.

    Returns A (len(rows), N) complex128, b (n_rhs, len(rows))."""
    o = _opts(opts)
    v = np.asarray(v, dtype=np.float64)
    t = np.asarray(t, dtype=np.int64)
    N = t.shape[0]
    rows = np.arange(N) if rows is None else np.asarray(rows)
    V1, V2, V3 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    c, nrm, area = geom["centroid"], geom["normal"], geom["area"]
    lam_f, w_f = quadrature.rule(o["far_pts"])
    lam_n, w_n = quadrature.composite_rule(o["near_levels_N"], 7)
    Yf = np.einsum("qa,mad->mqd", lam_f, np.stack([V1, V2, V3], axis=1))
    if near is None:
        near = nearlist.near_list(t, c, geom["diam"], o["near_eta"], rows=rows)
    rp, col, cls = near
    A = np.zeros((len(rows), N), dtype=np.complex128)
    Vm = np.zeros((len(rows), N), dtype=np.complex128)
    for r, i in enumerate(rows):
        Xi = quadrature.map_points(lam_f, V1[i], V2[i], V3[i])
        K, V = np.zeros(N, np.complex128), np.zeros(N, np.complex128)
        idx = np.arange(N)
        idx = idx[idx != i]
        K[idx], V[idx] = tensor_entries(Xi, w_f, area[i], Yf[idx], w_f, nrm[idx], area[idx], k)
        js, cl = col[rp[r]:rp[r + 1]], cls[rp[r]:rp[r + 1]]
        jn = js[cl == nearlist.CLS_N]
        if jn.size:
            Xn = quadrature.map_points(lam_n, V1[i], V2[i], V3[i])
            Yn = np.einsum("qa,mad->mqd", lam_n, np.stack([V1[jn], V2[jn], V3[jn]], axis=1))
            K[jn], V[jn] = tensor_entries(Xn, w_n, area[i], Yn, w_n, nrm[jn], area[jn], k)
        for j in list(js[cl == nearlist.CLS_S]) + [i]:
            K[j], V[j] = ss_entry(v, t[i], t[j], nrm[j], area[i], area[j], k, o["ss_order"])
        K[i] = 0.0   # flat triangle: (y - x) . n_i = 0
        A[r] = -K
        A[r, i] += 0.5 * area[i]
        Vm[r] = V
    b = None
    if g is not None:
        g = np.atleast_2d(np.asarray(g, dtype=np.complex128))
        b = -(Vm @ g.T).T
    return A, b
