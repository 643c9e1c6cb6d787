"""Row a12: listener points (oracle, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper samples theta, phi, r "within an enclosing sphere, with the radius
constrained to be 1.5 to 3 times the size of the bounding box radius".
Reading R-listen: the configs use the pixel-centred spherical shell grid
    theta_u = -pi + (u + 1/2) 2 pi / n_theta,  phi_v = (v + 1/2) pi / n_phi,
    r_w = R (r_lo + (r_hi - r_lo)(w + 1/2) / n_r),
    x = centre + r (sin phi cos theta, sin phi sin theta, cos phi),
point index ((w n_phi) + v) n_theta + u (theta fastest); r_lo = 1.5, r_hi = 3.
Pinned by tests/test_oracle_listeners.py (radii, angles, count, ordering).
"""
import numpy as np


def shell_grid(centre, R, n_theta, n_phi, n_r, r_lo=1.5, r_hi=3.0):
    u = np.arange(n_theta)
    v = np.arange(n_phi)
    w = np.arange(n_r)
    th = -np.pi + (u + 0.5) * 2 * np.pi / n_theta
    ph = (v + 0.5) * np.pi / n_phi
    r = R * (r_lo + (r_hi - r_lo) * (w + 0.5) / n_r)
    W, Vv, U = np.meshgrid(w, v, u, indexing="ij")
    rr, pp, tt = r[W].ravel(), ph[Vv].ravel(), th[U].ravel()
    d = np.stack([np.sin(pp) * np.cos(tt), np.sin(pp) * np.sin(tt), np.cos(pp)], axis=1)
    return np.asarray(centre, dtype=np.float64)[None, :] + rr[:, None] * d
