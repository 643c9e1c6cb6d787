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


def test_random_shell_uniform_in_volume():
    """Reading R-listen-rand: bounds, r^3 uniform (KS), isotropic directions (cos(phi)
    uniform on [-1, 1] by KS, azimuth uniform, mean direction ~ 0)."""
    from scipy import stats
    c = np.array([0.5, -1.0, 2.0])
    R, n = 0.7, 100_000
    x = listeners.random_shell(c, R, n, seed=20250606, stream_id=3)
    d = x - c
    r = np.linalg.norm(d, axis=1)
    assert np.all(r >= 1.5 * R * (1 - 1e-14)) and np.all(r <= 3.0 * R * (1 + 1e-14))
    q = ((r / R) ** 3 - 1.5 ** 3) / (3.0 ** 3 - 1.5 ** 3)        # uniform on [0, 1] if uniform in volume
    assert stats.kstest(q, "uniform").pvalue > 1e-3
    assert stats.kstest((r / R - 1.5) / 1.5, "uniform").pvalue < 1e-6  # NOT uniform in radius
    cosp = d[:, 2] / r
    assert stats.kstest((cosp + 1) / 2, "uniform").pvalue > 1e-3
    az = (np.arctan2(d[:, 1], d[:, 0]) + math.pi) / (2 * math.pi)
    assert stats.kstest(az, "uniform").pvalue > 1e-3
    m = (d / r[:, None]).mean(axis=0)
    assert np.all(np.abs(m) < 4.0 / math.sqrt(3 * n))


def test_random_shell_streams_are_distinct_and_reproducible():
    a = listeners.random_shell([0, 0, 0], 1.0, 1000, seed=1, stream_id=0)
    b = listeners.random_shell([0, 0, 0], 1.0, 1000, seed=1, stream_id=0)
    np.testing.assert_array_equal(a, b)
    for other in (listeners.random_shell([0, 0, 0], 1.0, 1000, seed=2, stream_id=0),
                  listeners.random_shell([0, 0, 0], 1.0, 1000, seed=1, stream_id=1)):
        assert np.max(np.abs(a - other)) > 0.5
    # prefix property: point t depends only on t (counter-based)
    np.testing.assert_array_equal(listeners.random_shell([0, 0, 0], 1.0, 10, seed=1), a[:10])
