"""Free-space Helmholtz kernel and its normal derivative (oracle, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

G(x, y)      = e^{ikr} / (4 pi r),  r = |x - y|
dG/dn_y(x,y) = -e^{ikr} / (4 pi r^2) (1 - ikr) dr/dn_y,
               dr/dn_y = (y - x) . n_y / r
dG/dn_x(x,y) = G'(r) dr/dn_x,  dr/dn_x = -(y - x) . n_x / r,  G'(r) = e^{ikr}(ikr - 1)/(4 pi r^2)
d2G/dn_x dn_y = e^{ikr}/(4 pi r^3) [ -(d.n_x)(d.n_y)(3 - 3ikr - k^2 r^2)/r^2 - (n_x.n_y)(ikr - 1) ],
               d = y - x  (the two normal derivatives of Eq. BM)
Time convention e^{+ikr} (outgoing), as the paper writes the kernel.
r < 1e-12 is a singular evaluation and raises.
Pinned by tests/test_oracle_kernel.py (worked values, reciprocity, |G| = 1/(4 pi r),
finite differences) and tests/test_oracle_bm.py (finite differences of the x-derivatives).
"""
import numpy as np

SINGULAR_R = 1e-12


def _dist(x, y):
    d = np.asarray(y, dtype=np.float64) - np.asarray(x, dtype=np.float64)
    r = np.sqrt(np.sum(d * d, axis=-1))
    if np.any(r < SINGULAR_R):
        raise ZeroDivisionError("singular kernel evaluation: |x - y| < 1e-12")
    return d, r


def green(x, y, k):
    """G(x, y) = e^{ikr}/(4 pi r).  Broadcasts over leading axes."""
    _, r = _dist(x, y)
    return np.exp(1j * k * r) / (4.0 * np.pi * r)


def green_dn_y(x, y, n_y, k):
    """dG/dn_y = -e^{ikr}/(4 pi r^2) (1 - ikr) dr/dn_y,  dr/dn_y = (y-x).n_y / r."""
    d, r = _dist(x, y)
    dr_dn = np.sum(d * np.asarray(n_y, dtype=np.float64), axis=-1) / r
    return -np.exp(1j * k * r) / (4.0 * np.pi * r * r) * (1.0 - 1j * k * r) * dr_dn


def green_dn_x(x, y, n_x, k):
    """dG/dn_x = G'(r) (x - y).n_x / r   (adjoint double-layer kernel of Eq. BM)."""
    d, r = _dist(x, y)
    dr_dn = -np.sum(d * np.asarray(n_x, dtype=np.float64), axis=-1) / r
    return np.exp(1j * k * r) * (1j * k * r - 1.0) / (4.0 * np.pi * r * r) * dr_dn


def green_dn_x_dn_y(x, y, n_x, n_y, k):
    """d^2 G / dn_x dn_y   (hypersingular kernel of Eq. BM, l.176)."""
    d, r = _dist(x, y)
    dnx = np.sum(d * np.asarray(n_x, dtype=np.float64), axis=-1)
    dny = np.sum(d * np.asarray(n_y, dtype=np.float64), axis=-1)
    nn = np.sum(np.asarray(n_x, dtype=np.float64) * np.asarray(n_y, dtype=np.float64), axis=-1)
    kr = k * r
    return np.exp(1j * kr) / (4.0 * np.pi * r ** 3) * (
        -dnx * dny * (3.0 - 3j * kr - kr * kr) / (r * r) - nn * (1j * kr - 1.0))
