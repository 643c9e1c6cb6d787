"""Row a11: radiation of the solved surface field to listener points (oracle, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

"computing the sound pressure at any point in space from the Neumann and Dirichlet
conditions".  Exterior representation formula with coefficient 1
(reading R-ext; the paper writes only the on-boundary 1/2 form, l.196):
    p(x) = int_Gamma [p(y) dG/dn_y(x,y) - g(y) G(x,y)] dS(y)
         ~ sum_s w_s [p_s dG/dn_y(x, y_s) - g_s G(x, y_s)].
Sources: BEM solution -> R3 quadrature points of every triangle, w = omega_q A_t,
normal n_t, values p_t, g_t;  MC solution -> the samples, w = |Gamma| / M.
Pinned by tests/test_oracle_radiate.py (pulsating sphere exterior field and the exact
interior extinction at the centre with analytic boundary data, interior point-source
reproduction, 1/r far-field decay).
"""
import numpy as np

from . import kernel, quadrature


def bem_sources(v, t, geom, p_tri, g_tri, q_rad=3):
    """Returns (y (3N... ,3), n, w, p (n_modes, S), g (n_modes, S))."""
    v = np.asarray(v, dtype=np.float64)
    t = np.asarray(t, dtype=np.int64)
    lam, wq = quadrature.rule(q_rad)
    V1, V2, V3 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    y = (lam[None, :, 0:1] * V1[:, None] + lam[None, :, 1:2] * V2[:, None]) \
        + lam[None, :, 2:3] * V3[:, None]
    Q = lam.shape[0]
    y = y.reshape(-1, 3)
    n = np.repeat(geom["normal"], Q, axis=0)
    w = (geom["area"][:, None] * wq[None, :]).reshape(-1)
    p = np.repeat(np.atleast_2d(p_tri), Q, axis=1)
    g = np.repeat(np.atleast_2d(g_tri), Q, axis=1)
    return y, n, w, p, g


def mc_sources(y, n, total_area, p, g):
    M = y.shape[0]
    return y, n, np.full(M, total_area / M), np.atleast_2d(p), np.atleast_2d(g)


def radiate(src, ks, x, chunk=256):
    """p[m, l] = sum_s w_s [p_ms dG_m/dn_y(x_l, y_s) - g_ms G_m(x_l, y_s)]."""
    y, n, w, p, g = src
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros((len(ks), x.shape[0]), np.complex128)
    for m, k in enumerate(ks):
        for a in range(0, x.shape[0], chunk):
            xl = x[a:a + chunk, None, :]
            dG = kernel.green_dn_y(xl, y[None], n[None], k)
            G = kernel.green(xl, y[None], k)
            out[m, a:a + chunk] = np.sum(w[None] * (p[m][None] * dG - g[m][None] * G), axis=1)
    return out
