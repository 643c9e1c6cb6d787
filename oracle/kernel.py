"""Free-space Helmholtz kernel and its normal derivative (oracle, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

G(x, y)      = e^{ikr} / (4 pi r),  r = |x - y|
dG/dn_y(x,y) = -e^{ikr} / (4 pi r^2) (1 - ikr) dr/dn_y,
               dr/dn_y = (y - x) . n_y / r
Time convention e^{+ikr} (outgoing), as the paper writes the kernel.
r < 1e-12 is a singular evaluation and raises.
Pinned by tests/test_oracle_kernel.py (worked values, reciprocity, |G| = 1/(4 pi r),
finite differences).
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
