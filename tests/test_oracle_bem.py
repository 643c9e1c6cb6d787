"""Pins of oracle.bem (rows a4-a6) against the mathematics: Gauss identity, sphere
eigenvalues, brute-force adaptive integrals, and the analytic sphere / point-source
solutions (north-star acceptance: <= 2%)."""
import functools

import numpy as np
import pytest
from scipy import integrate

import nat_inputs as I
from oracle import analytic, bem, geometry, gmres, kernel, listeners, nearlist, radiate


@functools.lru_cache(maxsize=None)
def _mesh(level):
    m = I.icosphere(level)
    geo = geometry.mesh_prepare(m.v, m.t)
    near = nearlist.near_list(m.t, geo["centroid"], geo["diam"])
    return m, geo, near


def test_gauss_identity_k0():
    # sum_j K_ij = -1/2 for a collocation point on a flat part of a closed surface,
    # so every row of A = 1/2 I - K sums to 1.
    m, geo, near = _mesh(3)
    A, _ = bem.assemble(m.v, m.t, geo, 0.0, None, near=near)
    assert np.max(np.abs(A.sum(axis=1) - 1.0)) < 1e-4


def test_sphere_eigenvalues_converge():
    errs = {}
    for L in (2, 3):
        m, geo, near = _mesh(L)
        d = geo["centroid"] / np.linalg.norm(geo["centroid"], axis=1, keepdims=True)
        Y = np.stack([np.ones(m.n_tri), d[:, 2], 1.5 * d[:, 2] ** 2 - 0.5]).astype(complex)
        k = 2.0
        A, b = bem.assemble(m.v, m.t, geo, k, Y, near=near)
        e = []
        for n in range(3):
            yy = np.vdot(Y[n], Y[n])
            lamK = 0.5 - np.vdot(Y[n], A @ Y[n]) / yy
            lamV = -np.vdot(Y[n], b[n]) / yy
            eK, eV = analytic.sphere_eig_K(n, k), analytic.sphere_eig_V(n, k)
            e.append(max(abs(lamK - eK) / abs(0.5 - eK), abs(lamV - eV) / abs(eV)))
        errs[L] = max(e)
    assert errs[2] < 0.04 and errs[3] < 0.01
    assert errs[2] / errs[3] > 3.0          # O(h^2)


def _brute(m, geo, i, j, k):
    v1, v2, v3 = m.v[m.t[j]]
    x, n, J = geo["centroid"][i], geo["normal"][j], 2 * geo["area"][j]

    def f(s, r, which, part):
        y = v1 + r * (v2 - v1) + s * (v3 - v1)
        val = kernel.green(x, y, k) if which == "V" else kernel.green_dn_y(x, y, n, k)
        return (val.real if part == 0 else val.imag) * J

    out = {}
    for which in ("V", "K"):
        re, im = (integrate.dblquad(f, 0, 1, 0, lambda r: 1 - r, args=(which, p),
                                    epsabs=1e-13, epsrel=1e-11)[0] for p in (0, 1))
        out[which] = re + 1j * im
    return out


def test_entries_vs_adaptive_integration():
    m, geo, near = _mesh(2)
    k = 2.0
    rows = [0, 77]
    rp, col, cls = nearlist.near_list(m.t, geo["centroid"], geo["diam"], rows=rows)
    A, _, V = bem.assemble(m.v, m.t, geo, k, None, rows=rows, near=(rp, col, cls),
                           return_V=True)
    for r, i in enumerate(rows):
        js, cs = col[rp[r]:rp[r + 1]], cls[rp[r]:rp[r + 1]]
        listed = set(js.tolist())
        far = [j for j in range(m.n_tri) if j not in listed and j != i]
        picks = [(js[cs == 1][0], 1e-5), (js[cs == 1][-1], 1e-5),
                 (js[cs == 2][0], 1e-5), (js[cs == 2][-1], 1e-5),
                 (far[0], 1e-3), (far[-1], 1e-3)]
        for j, tol in picks:
            ref = _brute(m, geo, i, j, k)
            assert abs(V[r, j] - ref["V"]) <= tol * abs(ref["V"])
            assert abs(-A[r, j] - ref["K"]) <= tol * abs(ref["K"])
        assert A[r, i] == 0.5


def _solve_field(level, k, g, L):
    m, geo, near = _mesh(level)
    A, b = bem.assemble(m.v, m.t, geo, k, g, near=near)
    out = []
    for r in range(b.shape[0]):
        x, info = gmres.gmres(lambda z: A @ z, b[r], tol=1e-12, max_iter=200)
        assert info["converged"] == 1
        src = radiate.bem_sources(m.v, m.t, geo, x[None], g[r][None])
        out.append((x, radiate.radiate(src, [k], L)[0]))
    return out


def test_c1_pulsating_sphere_within_2_percent():
    """Config C1: icosphere L3 (1280 tri), g = 1, k = 1, 4x4x4 shell grid."""
    m, geo, _ = _mesh(3)
    L = listeners.shell_grid(np.zeros(3), 1.0, 4, 4, 4)
    [(x, p)] = _solve_field(3, 1.0, I.neumann_constant(m)[None], L)
    pe = analytic.pulsating_sphere(np.linalg.norm(L, axis=1), 1.0)
    assert np.linalg.norm(p - pe) / np.linalg.norm(pe) < 0.02
    pb = analytic.pulsating_sphere(1.0, 1.0)
    assert np.sqrt(np.mean(np.abs(x - pb) ** 2)) / abs(pb) < 0.02


@pytest.mark.parametrize("k", [0.5, 2.0])
def test_oscillating_sphere_within_2_percent(k):
    m, geo, _ = _mesh(3)
    L = listeners.shell_grid(np.zeros(3), 1.0, 8, 8, 2)
    [(_, p)] = _solve_field(3, k, I.neumann_rigid_z(m)[None], L)
    pe = analytic.oscillating_sphere(L, k)
    assert np.linalg.norm(p - pe) / np.linalg.norm(pe) < 0.02


def test_interior_point_source_manufactured():
    """PAPER.md l.398 analytic test idea: Neumann data of an interior source; the
    solved exterior field must reproduce the source's free field."""
    m, geo, _ = _mesh(3)
    xs, k = np.array([0.1, 0.2, -0.1]), 1.0
    g = analytic.point_source_dn(geo["centroid"], geo["normal"], xs, k)
    L = listeners.shell_grid(np.zeros(3), 1.0, 4, 4, 4)
    [(x, p)] = _solve_field(3, k, g[None], L)
    pe = analytic.point_source(L, xs, k)
    assert np.linalg.norm(p - pe) / np.linalg.norm(pe) < 0.02
    pb = analytic.point_source(geo["centroid"], xs, k)
    assert np.linalg.norm(x - pb) / np.linalg.norm(pb) < 0.02


def _thin_wall_case(n_az, n_psi, k=2.0):
    """SURVEY §8(d) C3 acceptance (thin-wall sanity pin; the idea is P:398's analytic point
    source): x_s = (0, 0, -0.95) inside the 0.1-thick wall of the bowl, g_t = dG(c_t, x_s)/dn_t;
    the exterior field must approach G(x, x_s)."""
    m = I.bowl(n_az, n_psi, 2)
    geo = geometry.mesh_prepare(m.v, m.t)
    xs = np.array([0.0, 0.0, -0.95])
    g = analytic.point_source_dn(geo["centroid"], geo["normal"], xs, k)
    A, b = bem.assemble(m.v, m.t, geo, k, g[None])
    x, info = gmres.gmres(lambda z: A @ z, b[0], 1e-10, 400)
    L = listeners.shell_grid(geo["center"], geo["bound_radius"], 8, 8, 4)
    p = radiate.radiate(radiate.bem_sources(m.v, m.t, geo, x[None], g[None]), [k], L)[0]
    pe = analytic.point_source(L, xs, k)
    return np.linalg.norm(p - pe) / np.linalg.norm(pe)


def test_thin_wall_point_source_converges():
    """The source sits about one element from both faces of the wall, so P0 collocation is
    far from its 2% sphere accuracy on coarse bowls; the pin is convergence: the field
    error at 3,200 triangles is below 0.3 and below half of the 832-triangle error
    (measured: 0.60 -> 0.26).  The 12,544-triangle case runs on the GPU
    (tests/test_gpu_configs.py) with the tolerance set from these oracle errors."""
    e0 = _thin_wall_case(32, 6)
    e1 = _thin_wall_case(64, 12)
    assert e1 < 0.3 and e1 < 0.5 * e0
