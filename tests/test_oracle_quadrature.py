"""Pins of oracle.quadrature: rule exactness, subdivision, polar self term."""
import math

import numpy as np
import pytest
from scipy import integrate

from conftest import load_golden
from oracle import quadrature


def _monomial_exact(a, b):
    # int over the reference triangle (0,0),(1,0),(0,1) of x^a y^b = a! b! / (a+b+2)!
    return math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)


@pytest.mark.parametrize("npts,degree", [(1, 1), (3, 2), (6, 4), (7, 5)])
def test_rule_exactness(npts, degree):
    lam, w = quadrature.rule(npts)
    assert abs(w.sum() - 1) < 1e-15
    assert np.all(np.abs(lam.sum(axis=1) - 1) < 1e-15)
    x, y = lam[:, 1], lam[:, 2]
    for a in range(degree + 1):
        for b in range(degree + 1 - a):
            q = 0.5 * np.sum(w * x ** a * y ** b)
            assert abs(q - _monomial_exact(a, b)) < 1e-15


@pytest.mark.parametrize("level", [1, 2, 3])
def test_composite_rule(level):
    lam, w = quadrature.composite_rule(level, 7)
    assert lam.shape == (7 * 4 ** level, 3)
    assert abs(w.sum() - 1) < 1e-14
    x, y = lam[:, 1], lam[:, 2]
    for a in range(6):
        for b in range(6 - a):
            assert abs(0.5 * np.sum(w * x ** a * y ** b) - _monomial_exact(a, b)) < 1e-15
    # a non-polynomial integrand converges towards the adaptive value as level grows
    f = lambda x, y: np.sqrt(x + y + 0.01)
    ref = integrate.dblquad(lambda yy, xx: f(xx, yy), 0, 1, 0, lambda xx: 1 - xx,
                            epsabs=1e-13)[0]
    err = abs(0.5 * np.sum(w * f(x, y)) - ref)
    assert err < 5e-3 / 4 ** level


def _polar_adaptive(v1, v2, v3, k):
    """Independent: global polar angle about the centroid, R(theta) by ray/edge
    intersection, scipy adaptive quadrature of (e^{ikR}-1)/(4 pi i k) d theta."""
    c = (v1 + v2 + v3) / 3
    e1 = (v2 - v1) / np.linalg.norm(v2 - v1)
    nrm = np.cross(v2 - v1, v3 - v1)
    e2 = np.cross(nrm / np.linalg.norm(nrm), e1)
    P = [np.array([np.dot(p - c, e1), np.dot(p - c, e2)]) for p in (v1, v2, v3)]

    def R(th):
        d = np.array([math.cos(th), math.sin(th)])
        best = np.inf
        for a, b in ((P[0], P[1]), (P[1], P[2]), (P[2], P[0])):
            M = np.array([d, a - b]).T
            s, tt = np.linalg.solve(M, a)
            if s > 0 and -1e-12 <= tt <= 1 + 1e-12:
                best = min(best, s)
        return best

    def f(th, part):
        r = R(th)
        val = r if k == 0 else (np.exp(1j * k * r) - 1) / (1j * k)
        return (val.real if part == 0 else val.imag) if k else (val if part == 0 else 0.0)

    brk = sorted(math.atan2(p[1], p[0]) % (2 * math.pi) for p in P)
    out = 0j
    for part in (0, 1):
        s = integrate.quad(f, 0, 2 * math.pi, args=(part,), points=brk, epsabs=1e-14,
                           epsrel=1e-13, limit=200)[0]
        out += s if part == 0 else 1j * s
    return out / (4 * math.pi)


def test_self_term_golden_equilateral():
    v1 = np.array([0.0, 0.0, 0.0])
    v2 = np.array([1.0, 0.0, 0.0])
    v3 = np.array([0.5, math.sqrt(3) / 2, 0.0])
    for k, re, im, tol in load_golden("self_term.txt"):
        k, re, im, tol = map(float, (k, re, im, tol))
        val = quadrature.self_single_layer(v1, v2, v3, k)
        assert abs(val - (re + 1j * im)) < tol
    assert abs(quadrature.self_single_layer(v1, v2, v3, 0.0)
               - math.sqrt(3) * math.log(2 + math.sqrt(3)) / (4 * math.pi)) < 1e-13


def test_self_term_vs_closed_form_and_adaptive():
    rng = np.random.default_rng(5)
    for _ in range(6):
        v = rng.normal(size=(3, 3))
        # avoid extreme slivers so GL16 per edge is converged
        e = np.cross(v[1] - v[0], v[2] - v[0])
        if np.linalg.norm(e) < 0.3:
            continue
        k0 = quadrature.self_single_layer(v[0], v[1], v[2], 0.0)
        assert abs(k0 - quadrature.self_single_layer_k0_closed(*v)) < 1e-7 * abs(k0)
        assert abs(k0 - _polar_adaptive(*v, 0.0)) < 1e-7 * abs(k0)
        diam = max(np.linalg.norm(v[a] - v[b]) for a, b in ((0, 1), (1, 2), (2, 0)))
        for kd in (0.5, 3.0):   # k * diam: the BEM configs stay below ~1
            k = kd / diam
            val = quadrature.self_single_layer(v[0], v[1], v[2], k)
            ref = _polar_adaptive(*v, k)
            assert abs(val - ref) < 5e-7 * abs(ref)   # GL16-per-edge rule error


def test_self_term_small_k_expansion():
    # V(k) = V(0) + ik A/(4 pi) + O(k^2)  (expand e^{ik rho} = 1 + ik rho + ...)
    v1, v2, v3 = np.array([0., 0, 0]), np.array([0.3, 0, 0]), np.array([0.1, 0.25, 0])
    A = 0.5 * np.linalg.norm(np.cross(v2 - v1, v3 - v1))
    V0 = quadrature.self_single_layer(v1, v2, v3, 0.0)
    for k in (1e-3, 1e-2):
        Vk = quadrature.self_single_layer(v1, v2, v3, k)
        assert abs(Vk - (V0 + 1j * k * A / (4 * math.pi))) < 2 * k * k * A * 0.3
