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

The optional random form (reading R-listen-rand, SPEC's "uniform in volume" note to
P:166): point t draws (o0..o3) = Philox4x32-10(counter (t, 1, stream_lo, stream_hi),
key = seed), u_a = (o_a + 1/2) 2^-32, and sets cos(phi) = 1 - 2 u0 (uniform direction),
sin(phi) = 2 sqrt(u0 (1 - u0)), theta = -pi + 2 pi u1, r = R cbrt(r_lo^3 + u2 (r_hi^3 -
r_lo^3)) (uniform in volume).  Pinned by tests/test_oracle_listeners.py (bounds,
Kolmogorov-Smirnov of r^3 and of cos(phi), isotropy, seed/stream/tag independence).
"""
import numpy as np

from . import philox


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


def random_shell(centre, R, n, r_lo=1.5, r_hi=3.0, seed=0, stream_id=0):
    t = np.arange(n, dtype=np.uint64)
    u = philox.uniforms(t, tag=1, stream_id=stream_id, seed=seed)   # (n, 4) fp64 in (0, 1)
    u0, u1, u2 = u[:, 0], u[:, 1], u[:, 2]
    cp = 1.0 - 2.0 * u0
    sp = 2.0 * np.sqrt(u0 * (1.0 - u0))
    th = -np.pi + 2.0 * np.pi * u1
    lo3, hi3 = r_lo ** 3, r_hi ** 3
    r = R * np.cbrt(lo3 + u2 * (hi3 - lo3))
    d = np.stack([sp * np.cos(th), sp * np.sin(th), cp], axis=1)
    return np.asarray(centre, dtype=np.float64)[None, :] + r[:, None] * d
