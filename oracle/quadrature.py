"""Triangle quadrature, subdivision and the polar self term (oracle, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper integrates element pairs with "Gaussian quadrature" and treats "adjacent or
identical elements" specially without giving the rules; the rules
here are the build's reading R-quad of DESIGN.md §3:

  R1  1 point,  degree 1:  (1/3,1/3,1/3), w = 1
  R3  3 points, degree 2:  permutations of (2/3,1/6,1/6), w = 1/3
  R6  6 points, degree 4:  Strang-Fix / Dunavant
  R7  7 points, degree 5:  Radon: centroid 9/40; (1-2a, a, a), a = (6 -+ sqrt15)/21,
                           w = (155 -+ sqrt15)/1200
  subdivision: (v1,v2,v3) -> (v1,m12,m13), (m12,v2,m23), (m13,m23,v3), (m12,m23,m13)

Self term (collocation point at the centroid of its own flat triangle).  The paper's
disk argument integrates G in polar coordinates about the
singular point, int_0^R e^{ik rho}/(4 pi rho) rho d rho = (e^{ikR}-1)/(4 pi i k); here
it is applied exactly over the triangle instead of a disk: with h_e the distance from
the centroid to edge e and alpha the polar angle measured from the foot of the
perpendicular, R(alpha) = h_e / cos(alpha) and
  V_ii = 1/(4 pi) sum_e int_{alpha_e0}^{alpha_e1} R E(kR) d alpha,
  E(x) = (e^{ix} - 1)/(ix) = sin(x)/x + i (1 - cos x)/x     (E(0) = 1).
With the substitution tan(alpha) = sinh(u) (s = h sinh u along the edge) this is
  V_ii = 1/(4 pi) sum_e h_e int_{u_e0}^{u_e1} E(k h_e cosh u) du,  u = asinh(s / h_e),
whose integrand is entire and exactly constant at k = 0; it is integrated with
Gauss-Legendre (16 points per edge) in u (reading R-self).  K_ii = 0 exactly because
(y - c_i) . n_i = 0 on a flat triangle (the perpendicularity argument of PAPER.md
l.233-236 holds exactly here).
Pinned by tests/test_oracle_quadrature.py: weights/exactness on monomials, the k = 0
closed form h[asinh(s1/h) - asinh(s0/h)], the equilateral value, adaptive polar
integration for k > 0, and the paper-free small-k expansion.
"""
import math

import numpy as np

_SQ15 = math.sqrt(15.0)


def rule(npts: int):
    """Barycentric points (Q,3) and weights (Q,) summing to 1."""
    if npts == 1:
        return np.array([[1 / 3, 1 / 3, 1 / 3]]), np.array([1.0])
    if npts == 3:
        p = np.array([[2 / 3, 1 / 6, 1 / 6], [1 / 6, 2 / 3, 1 / 6], [1 / 6, 1 / 6, 2 / 3]])
        return p, np.full(3, 1 / 3)
    if npts == 6:
        a1, b1, w1 = 0.10810301816807023, 0.44594849091596489, 0.22338158967801147
        a2, b2, w2 = 0.81684757298045851, 0.091576213509770743, 0.10995174365532187
        p = np.array([[a1, b1, b1], [b1, a1, b1], [b1, b1, a1],
                      [a2, b2, b2], [b2, a2, b2], [b2, b2, a2]])
        return p, np.array([w1] * 3 + [w2] * 3)
    if npts == 7:
        ap, am = (6 + _SQ15) / 21, (6 - _SQ15) / 21
        wp, wm = (155 + _SQ15) / 1200, (155 - _SQ15) / 1200
        p = [[1 / 3, 1 / 3, 1 / 3]]
        w = [9 / 40]
        for a, wa in ((ap, wp), (am, wm)):
            b = 1 - 2 * a
            p += [[b, a, a], [a, b, a], [a, a, b]]
            w += [wa] * 3
        return np.array(p), np.array(w)
    raise ValueError(f"no {npts}-point rule")


def subdivide(level: int):
    """Barycentric vertex triples (S,3,3) of the 4^level midpoint subtriangles."""
    tris = [np.eye(3)]
    for _ in range(level):
        nxt = []
        for p in tris:
            m12, m13, m23 = (p[0] + p[1]) / 2, (p[0] + p[2]) / 2, (p[1] + p[2]) / 2
            nxt += [np.array([p[0], m12, m13]), np.array([m12, p[1], m23]),
                    np.array([m13, m23, p[2]]), np.array([m12, m23, m13])]
        tris = nxt
    return np.array(tris)


def composite_rule(level: int, npts: int):
    """Rule ``npts`` on each of the 4^level subtriangles, expressed in the parent's
    barycentric coordinates; weights sum to 1."""
    p, w = rule(npts)
    sub = subdivide(level)
    pts = np.einsum("qa,sab->sqb", p, sub).reshape(-1, 3)
    wts = np.tile(w, len(sub)) / len(sub)
    return pts, wts


def map_points(lam, v1, v2, v3):
    """Physical points (lam1 v1 + lam2 v2) + lam3 v3 for barycentrics lam (Q,3)."""
    return (lam[:, 0:1] * v1 + lam[:, 1:2] * v2) + lam[:, 2:3] * v3


def _E(x):
    """(e^{ix} - 1)/(ix), stable for small x."""
    x = np.asarray(x, dtype=np.float64)
    out = np.ones_like(x, dtype=np.complex128)
    nz = x != 0
    xs = x[nz]
    out[nz] = np.sin(xs) / xs + 1j * (2.0 * np.sin(xs / 2) ** 2) / xs
    return out


def self_single_layer(v1, v2, v3, k, n_gl: int = 16, point=None):
    """V_ii = int_T G(c, y) dS(y) with c the centroid (or ``point``, inside T)."""
    v1, v2, v3 = (np.asarray(a, dtype=np.float64) for a in (v1, v2, v3))
    c = ((v1 + v2) + v3) / 3.0 if point is None else np.asarray(point, dtype=np.float64)
    xg, wg = np.polynomial.legendre.leggauss(n_gl)
    total = 0.0 + 0.0j
    for a, b in ((v1, v2), (v2, v3), (v3, v1)):
        L = np.linalg.norm(b - a)
        u = (b - a) / L
        foot = a + np.dot(c - a, u) * u
        h = np.linalg.norm(c - foot)
        s0, s1 = np.dot(a - foot, u), np.dot(b - foot, u)
        u0, u1 = math.asinh(s0 / h), math.asinh(s1 / h)
        half, mid = (u1 - u0) / 2, (u1 + u0) / 2
        u = mid + half * xg
        R = h * np.cosh(u)
        total += h * np.sum(wg * half * _E(k * R))
    return total / (4.0 * np.pi)


def self_single_layer_k0_closed(v1, v2, v3):
    """k = 0 closed form (1/4pi) sum_e h_e [asinh(s1/h) - asinh(s0/h)] at the centroid."""
    v1, v2, v3 = (np.asarray(a, dtype=np.float64) for a in (v1, v2, v3))
    c = (v1 + v2 + v3) / 3.0
    tot = 0.0
    for a, b in ((v1, v2), (v2, v3), (v3, v1)):
        u = (b - a) / np.linalg.norm(b - a)
        foot = a + np.dot(c - a, u) * u
        h = np.linalg.norm(c - foot)
        s0, s1 = np.dot(a - foot, u), np.dot(b - foot, u)
        tot += h * (math.asinh(s1 / h) - math.asinh(s0 / h))
    return tot / (4.0 * np.pi)


def self_hypersingular(v1, v2, v3, k, n_gl: int = 16):
    """W_ii = f.p. int_T d2G/dn_x dn_y(c, y) dS(y) at the centroid c of the flat triangle
    (reading R-bm-self): there d.n_x = d.n_y = 0 and n_x.n_y = 1, so the integrand is
    e^{ikr}(1 - ikr)/(4 pi r^3); in polar coordinates about c, with
    int_0^R e^{ik rho}(1 - ik rho)/rho^2 d rho = [-e^{ik rho}/rho], the Hadamard finite part is
        W_ii = ik/2 - (1/4pi) oint e^{ik R(theta)} / R(theta) d theta,
    and per edge (distance h_e, s = h sinh u along the edge) d theta / R = du / (h cosh^2 u):
        W_ii = ik/2 - (1/4pi) sum_e (1/h_e) int e^{ik h_e cosh u} / cosh^2 u du   (GL n_gl in u)."""
    v1, v2, v3 = (np.asarray(a, dtype=np.float64) for a in (v1, v2, v3))
    c = ((v1 + v2) + v3) / 3.0
    xg, wg = np.polynomial.legendre.leggauss(n_gl)
    total = 0.0 + 0.0j
    for a, b in ((v1, v2), (v2, v3), (v3, v1)):
        L = np.linalg.norm(b - a)
        e = (b - a) / L
        foot = a + np.dot(c - a, e) * e
        h = np.linalg.norm(c - foot)
        s0, s1 = np.dot(a - foot, e), np.dot(b - foot, e)
        u0, u1 = math.asinh(s0 / h), math.asinh(s1 / h)
        half, mid = (u1 - u0) / 2, (u1 + u0) / 2
        u = mid + half * xg
        ch = np.cosh(u)
        total += np.sum(wg * half * np.exp(1j * k * h * ch) / (ch * ch)) / h
    return 0.5j * k - total / (4.0 * np.pi)


def self_hypersingular_k0_closed(v1, v2, v3):
    """k = 0: W_ii = -(1/4pi) sum_e (sin a1 - sin a0)/h_e, sin a = s / sqrt(s^2 + h^2)."""
    v1, v2, v3 = (np.asarray(a, dtype=np.float64) for a in (v1, v2, v3))
    c = (v1 + v2 + v3) / 3.0
    tot = 0.0
    for a, b in ((v1, v2), (v2, v3), (v3, v1)):
        e = (b - a) / np.linalg.norm(b - a)
        foot = a + np.dot(c - a, e) * e
        h = np.linalg.norm(c - foot)
        s0, s1 = np.dot(a - foot, e), np.dot(b - foot, e)
        tot += (s1 / math.hypot(s1, h) - s0 / math.hypot(s0, h)) / h
    return -tot / (4.0 * np.pi)
