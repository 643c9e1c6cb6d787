"""Pins of oracle.kernel (G, dG/dn_y) — no GPU."""
import numpy as np
import pytest

from conftest import load_golden
from oracle import kernel


def test_worked_values():
    for which, r, k, drdn, re, im, tol in load_golden("kernel_values.txt"):
        r, k, drdn, re, im, tol = map(float, (r, k, drdn, re, im, tol))
        x = np.zeros(3)
        y = np.array([r, 0.0, 0.0])
        if which == "green":
            val = kernel.green(x, y, k)
        else:
            n = np.array([drdn, np.sqrt(max(0.0, 1 - drdn ** 2)), 0.0])
            val = kernel.green_dn_y(x, y, n, k)
        assert abs(val - (re + 1j * im)) < tol


def test_perpendicular_normal_is_exact_zero():
    x = np.array([0.3, -0.2, 0.1])
    y = x + np.array([0.0, 0.7, 0.0])
    n = np.array([1.0, 0.0, 0.0])
    for k in (0.0, 1.0, 37.0):
        assert kernel.green_dn_y(x, y, n, k) == 0.0


def test_singular_raises():
    x = np.array([0.1, 0.2, 0.3])
    with pytest.raises(ZeroDivisionError):
        kernel.green(x, x, 1.0)
    with pytest.raises(ZeroDivisionError):
        kernel.green_dn_y(x, x, np.array([0, 0, 1.0]), 1.0)


def test_reciprocity_bitwise_and_modulus():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(10000, 3))
    y = rng.normal(size=(10000, 3))
    k = rng.uniform(0, 50, size=10000)
    a = kernel.green(x, y, k)
    b = kernel.green(y, x, k)
    assert np.array_equal(a, b)
    r = np.linalg.norm(x - y, axis=1)
    np.testing.assert_allclose(np.abs(a), 1 / (4 * np.pi * r), rtol=1e-13)


def test_normal_derivative_matches_finite_differences():
    rng = np.random.default_rng(2)
    for _ in range(200):
        r = rng.uniform(0.1, 10)
        k = rng.uniform(0, 50)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        x = rng.normal(size=3)
        y = x + r * d
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        h = 1e-4 / (k + 1 / r)
        fd = (kernel.green(x, y + h * n, k) - kernel.green(x, y - h * n, k)) / (2 * h)
        an = kernel.green_dn_y(x, y, n, k)
        scale = abs(kernel.green(x, y, k)) * (k + 1 / r)
        assert abs(fd - an) <= 1e-6 * scale
