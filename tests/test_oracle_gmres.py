"""Pins of oracle.gmres (row a7)."""
import numpy as np

from oracle import gmres


def _system(n, seed):
    rng = np.random.default_rng(seed)
    A = np.eye(n) + 0.3 * (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    return A, b


def test_matches_direct_solve():
    A, b = _system(200, 1)
    x, info = gmres.gmres(lambda z: A @ z, b, tol=1e-12, max_iter=200)
    assert info["converged"] == 1 and info["rel_residual"] <= 1e-11
    xe = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xe) / np.linalg.norm(xe) < 1e-11


def test_zero_rhs_and_nonconvergence():
    A, b = _system(50, 2)
    x, info = gmres.gmres(lambda z: A @ z, np.zeros(50, complex))
    assert info["iters"] == 0 and np.all(x == 0)
    x, info = gmres.gmres(lambda z: A @ z, b, tol=1e-14, max_iter=3)
    assert info["converged"] == 0 and info["iters"] == 3
    # best iterate of the 3-dim Krylov space: residual below the initial one
    assert info["rel_residual"] < 1.0


def test_exact_in_n_steps_for_small_system():
    A, b = _system(6, 3)
    x, info = gmres.gmres(lambda z: A @ z, b, tol=1e-13, max_iter=6)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12
