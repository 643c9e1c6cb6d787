"""Pins of oracle.listeners (row a12)."""
import math

import numpy as np

from oracle import listeners


def test_shell_grid_layout():
    c = np.array([0.1, -0.2, 0.3])
    R = 2.0
    x = listeners.shell_grid(c, R, 8, 4, 3)
    assert x.shape == (96, 3)
    d = x - c
    r = np.linalg.norm(d, axis=1)
    rw = R * (1.5 + 1.5 * (np.arange(3) + 0.5) / 3)
    np.testing.assert_allclose(r, np.repeat(rw, 32), rtol=1e-14)
    assert np.all(r >= 1.5 * R) and np.all(r <= 3 * R)
    # theta fastest: first 8 points share phi and r, theta = -pi + (u + 1/2) pi/4
    th = np.arctan2(d[:8, 1], d[:8, 0])
    np.testing.assert_allclose(np.unwrap(th), -math.pi + (np.arange(8) + 0.5) * math.pi / 4,
                               atol=1e-14)
    ph = np.arccos(d[::8, 2] / r[::8])[:4]
    np.testing.assert_allclose(ph, (np.arange(4) + 0.5) * math.pi / 4, atol=1e-14)
