"""Closed-form solutions used only as pins of the oracle (no discretisation).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Pulsating sphere (radius a, dp/dn = g):  p(r) = g a^2 e^{ik(r-a)} / ((ika - 1) r)
  (= g h0(kr) / (k h0'(ka))).
* Oscillating sphere (dp/dn = g0 cos theta): p = g0 a^3 cos(theta) e^{ik(r-a)} (ikr - 1)
  / (r^2 (2 - 2ika - k^2 a^2))  (= g0 h1(kr) cos(theta)/(k h1'(ka))).
* Point source at x_s: G(x, x_s) and its normal derivative at x, written with dG/dr =
  e^{ikr}(ikr - 1)/(4 pi r^2) — the interior manufactured solution of PAPER.md l.398
  ("three dipole sound sources positioned ... within a mesh").
* Sphere eigenvalues of the single and double layer on Y_n (outward normal):
  lambda_V = i k a^2 j_n(ka) h_n(ka),  lambda_K = 1/2 + i k^2 a^2 j_n(ka) h_n'(ka)
  (SURVEY.md Appendix B.1/C.4), h_n = j_n + i y_n.
"""
import numpy as np
from scipy.special import spherical_jn, spherical_yn


def pulsating_sphere(r, k, a=1.0, g=1.0):
    r = np.asarray(r, dtype=np.float64)
    return g * a * a * np.exp(1j * k * (r - a)) / ((1j * k * a - 1.0) * r)


def oscillating_sphere(x, k, a=1.0, g0=1.0):
    """x: (P,3) points about the origin, axis z."""
    x = np.asarray(x, dtype=np.float64)
    r = np.linalg.norm(x, axis=-1)
    cth = x[..., 2] / r
    return g0 * a ** 3 * cth * np.exp(1j * k * (r - a)) * (1j * k * r - 1.0) / (
        r * r * (2.0 - 2j * k * a - k * k * a * a))


def h_n(n, z, derivative=False):
    return spherical_jn(n, z, derivative) + 1j * spherical_yn(n, z, derivative)


def pulsating_sphere_hankel(r, k, a=1.0, g=1.0):
    return g * h_n(0, k * np.asarray(r)) / (k * h_n(0, k * a, True))


def oscillating_sphere_hankel(x, k, a=1.0, g0=1.0):
    x = np.asarray(x, dtype=np.float64)
    r = np.linalg.norm(x, axis=-1)
    return g0 * h_n(1, k * r) * (x[..., 2] / r) / (k * h_n(1, k * a, True))


def point_source(x, xs, k):
    d = np.asarray(x, dtype=np.float64) - np.asarray(xs, dtype=np.float64)
    r = np.linalg.norm(d, axis=-1)
    return np.exp(1j * k * r) / (4 * np.pi * r)


def point_source_dn(x, n, xs, k):
    """d/dn_x of e^{ik|x - xs|}/(4 pi |x - xs|) at x along n."""
    d = np.asarray(x, dtype=np.float64) - np.asarray(xs, dtype=np.float64)
    r = np.linalg.norm(d, axis=-1)
    dGdr = np.exp(1j * k * r) * (1j * k * r - 1.0) / (4 * np.pi * r * r)
    return dGdr * np.sum(d * np.asarray(n), axis=-1) / r


def sphere_eig_V(n, k, a=1.0):
    if k == 0:
        return a / (2 * n + 1)
    ka = k * a
    return 1j * k * a * a * spherical_jn(n, ka) * h_n(n, ka)


def sphere_eig_K(n, k, a=1.0):
    if k == 0:
        return -1.0 / (2 * (2 * n + 1))
    ka = k * a
    return 0.5 + 1j * k * k * a * a * spherical_jn(n, ka) * h_n(n, ka, True)
