"""Pins of oracle.galerkin (NEXT-2, reading R-galerkin) against the mathematics:
Sauter-Schwab cube maps integrate separable monomials over tau x tau exactly; the k = 0
single layer of coplanar identical / edge / vertex pairs equals the closed-form in-plane
potential of the source triangle integrated over the test triangle; the k > 0 part by
singularity subtraction; the Gauss identity of the Galerkin double layer; brute-force
far entries; the analytic pulsating / oscillating sphere within 2 %."""
import functools
import math

import numpy as np
import pytest

import nat_inputs as I
from oracle import analytic, galerkin, geometry, kernel, listeners, nearlist, quadrature, radiate


def _tau_monomial(a, b):
    # int_{0 <= x2 <= x1 <= 1} x1^a x2^b = 1 / ((b + 1)(a + b + 2))
    return 1.0 / ((b + 1) * (a + b + 2))


@pytest.mark.parametrize("case", ["identical", "edge", "vertex"])
def test_ss_rules_integrate_monomials_exactly(case):
    xh, yh, w = galerkin.ss_rule(case, 5)
    assert abs(w.sum() - 0.25) < 1e-15
    assert np.all(xh >= 0) and np.all(xh[:, 1] <= xh[:, 0] + 1e-15) and np.all(xh[:, 0] <= 1)
    assert np.all(yh >= 0) and np.all(yh[:, 1] <= yh[:, 0] + 1e-15) and np.all(yh[:, 0] <= 1)
    for a, b, c, d in [(1, 0, 0, 0), (0, 1, 2, 0), (2, 1, 1, 1), (1, 2, 0, 3), (0, 0, 2, 2)]:
        val = np.sum(w * xh[:, 0] ** a * xh[:, 1] ** b * yh[:, 0] ** c * yh[:, 1] ** d)
        assert abs(val - _tau_monomial(a, b) * _tau_monomial(c, d)) < 1e-15


def _inplane_potential(x, a, b, c):
    """int_T 1/|x - y| dS_y for x in the plane of T = (a, b, c): sum over the edges of the
    signed triangles (x, edge): d_e [asinh(s1/|d_e|) - asinh(s0/|d_e|)], d_e the signed
    distance of x to the edge line (positive on T's side)."""
    tot = 0.0
    cen = (a + b + c) / 3.0
    for p, q in ((a, b), (b, c), (c, a)):
        u = (q - p) / np.linalg.norm(q - p)
        foot = p + np.dot(x - p, u) * u
        dv = x - foot
        inward = cen - (p + np.dot(cen - p, u) * u)
        dist = np.linalg.norm(dv)
        if dist < 1e-300:
            continue
        sgn = 1.0 if np.dot(dv, inward) > 0 else -1.0
        s0, s1 = np.dot(p - foot, u), np.dot(q - foot, u)
        tot += sgn * dist * (math.asinh(s1 / dist) - math.asinh(s0 / dist))
    return tot


def _outer(fn, a, b, c, level=5):
    lam, w = quadrature.composite_rule(level, 7)
    pts = quadrature.map_points(lam, a, b, c)
    area = 0.5 * np.linalg.norm(np.cross(b - a, c - a))
    return area * sum(wq * fn(p) for p, wq in zip(pts, w))


# coplanar pairs in z = 0: (T_i, T_j) as vertex arrays and index triples
_P = np.array([[0.0, 0.0, 0.0], [1.0, 0.1, 0.0], [0.3, 0.9, 0.0], [1.2, 1.1, 0.0], [-0.8, -0.3, 0.0],
               [-0.2, -1.0, 0.0]])
_PAIRS = {"identical": ((0, 1, 2), (0, 1, 2)), "edge": ((0, 1, 2), (1, 3, 2)), "vertex": ((0, 1, 2), (0, 4, 5))}


@pytest.mark.parametrize("case", ["identical", "edge", "vertex"])
def test_ss_single_layer_k0_against_inplane_potential(case):
    ti, tj = _PAIRS[case]
    ai, aj = (0.5 * np.linalg.norm(np.cross(_P[t[1]] - _P[t[0]], _P[t[2]] - _P[t[0]])) for t in (ti, tj))
    nj = np.array([0.0, 0.0, 1.0])
    # the outer rule converges O(h^2) (the potential has x log x edge behaviour):
    # Richardson-extrapolate levels 5 and 6
    r5, r6 = (_outer(lambda x: _inplane_potential(x, *_P[list(tj)]), *_P[list(ti)], level=L) / (4 * np.pi)
              for L in (5, 6))
    ref = r6 + (r6 - r5) / 3.0
    K, V = galerkin.ss_entry(_P, ti, tj, nj, ai, aj, 0.0, 8)
    assert abs(K) < 1e-15                       # coplanar: (y - x) . n_j = 0
    assert abs(V - ref) / abs(ref) < 2e-7
    _, V4 = galerkin.ss_entry(_P, ti, tj, nj, ai, aj, 0.0, 4)   # the default order
    assert abs(V4 - ref) / abs(ref) < 2e-3


@pytest.mark.parametrize("case", ["identical", "edge", "vertex"])
def test_ss_single_layer_k3_by_singularity_subtraction(case):
    """G = 1/(4 pi r) + (e^{ikr} - 1)/(4 pi r): the second part is smooth (bounded by
    k/4pi), integrated by a converged tensor rule; the first by the in-plane potential."""
    k = 3.0
    ti, tj = _PAIRS[case]
    A, B = _P[list(ti)], _P[list(tj)]
    ai, aj = (0.5 * np.linalg.norm(np.cross(T[1] - T[0], T[2] - T[0])) for T in (A, B))
    r5, r6 = (_outer(lambda x: _inplane_potential(x, *B), *A, level=L) / (4 * np.pi) for L in (5, 6))
    sing = r6 + (r6 - r5) / 3.0
    sm = []
    for L in (3, 4):   # (cos kr - 1)/r ~ -k^2 r/2 has a kink on x = y: O(h^3), Richardson
        lam, w = quadrature.composite_rule(L, 7)
        X, Y = quadrature.map_points(lam, *A), quadrature.map_points(lam, *B)
        r = np.linalg.norm(X[:, None, :] - Y[None, :, :], axis=-1)
        safe = np.where(r > 0, r, 1.0)
        smooth = np.where(r > 0, (np.exp(1j * k * safe) - 1.0) / (4 * np.pi * safe), 1j * k / (4 * np.pi))
        sm.append(ai * aj * np.einsum("a,b,ab->", w, w, smooth))
    ref = sing + sm[1] + (sm[1] - sm[0]) / 7.0
    _, V = galerkin.ss_entry(_P, ti, tj, np.array([0, 0, 1.0]), ai, aj, k, 8)
    assert abs(V - ref) / abs(ref) < 2e-7


@functools.lru_cache(maxsize=None)
def _mesh(level):
    m = I.icosphere(level)
    geo = geometry.mesh_prepare(m.v, m.t)
    near = nearlist.near_list(m.t, geo["centroid"], geo["diam"])
    return m, geo, near


def test_gauss_identity_galerkin_k0():
    """sum_j int_{T_i} int_{T_j} dG0/dn_y = -|T_i| / 2 on a closed polyhedron (the solid
    angle seen from a face point is 2 pi); adjacent non-coplanar pairs carry most of it."""
    m, geo, near = _mesh(2)
    A, _ = galerkin.assemble(m.v, m.t, geo, 0.0, near=near)
    area = geo["area"]
    # A = 1/2 diag(|T|) - K  =>  row sums = |T_i| (1/2 + 1/2)
    assert np.max(np.abs(A.sum(axis=1) / area - 1.0)) < 2e-3
    # the Sauter-Schwab class-S entries alone are not small: the identity is not trivial
    rp, col, cls = near
    j = col[rp[0]:rp[1]][cls[rp[0]:rp[1]] == nearlist.CLS_S]
    assert np.abs(A[0, j]).sum() / area[0] > 0.05


def test_far_entries_brute_force():
    """Far-rule entries (R3 x R3) against a converged tensor rule on a separated pair; and
    the class-N rule (28 x 28) likewise on a close pair."""
    m, geo, near = _mesh(2)
    k = 2.0
    A, b = galerkin.assemble(m.v, m.t, geo, k, np.ones((1, m.n_tri)), rows=[5], near=None)
    rp, col, cls = nearlist.near_list(m.t, geo["centroid"], geo["diam"], rows=[5])
    far_j = [j for j in range(m.n_tri) if j != 5 and j not in set(col)]
    n_j = [j for j, c in zip(col, cls) if c == nearlist.CLS_N]
    lam, w = quadrature.composite_rule(3, 7)
    vi = m.v[m.t[5]]
    X = quadrature.map_points(lam, *vi)
    for j, tol in ((far_j[0], 2e-2), (far_j[len(far_j) // 2], 2e-3), (n_j[0], 1e-5)):
        vj = m.v[m.t[j]]
        Y = quadrature.map_points(lam, *vj)
        dG = kernel.green_dn_y(X[:, None, :], Y[None, :, :], geo["normal"][j][None, None, :], k)
        K = geo["area"][5] * geo["area"][j] * np.einsum("a,b,ab->", w, w, dG)
        assert abs(-A[0, j] - K) <= tol * abs(K)


def _galerkin_field(level, k, g, L):
    m, geo, near = _mesh(level)
    A, b = galerkin.assemble(m.v, m.t, geo, k, g[None], near=near)
    x = np.linalg.solve(A, b[0])
    src = radiate.bem_sources(m.v, m.t, geo, x[None], g[None])
    return x, radiate.radiate(src, [k], L)[0]


def test_galerkin_pulsating_sphere_within_2_percent():
    m, _, _ = _mesh(3)
    L = listeners.shell_grid(np.zeros(3), 1.0, 4, 4, 4)
    x, p = _galerkin_field(3, 1.0, I.neumann_constant(m), L)
    pe = analytic.pulsating_sphere(np.linalg.norm(L, axis=1), 1.0)
    assert np.linalg.norm(p - pe) / np.linalg.norm(pe) < 0.02
    pb = analytic.pulsating_sphere(1.0, 1.0)
    assert np.sqrt(np.mean(np.abs(x - pb) ** 2)) / abs(pb) < 0.02


def test_galerkin_oscillating_sphere_within_2_percent():
    m, _, _ = _mesh(3)
    L = listeners.shell_grid(np.zeros(3), 1.0, 8, 8, 2)
    _, p = _galerkin_field(3, 2.0, I.neumann_rigid_z(m), L)
    pe = analytic.oscillating_sphere(L, 2.0)
    assert np.linalg.norm(p - pe) / np.linalg.norm(pe) < 0.02
