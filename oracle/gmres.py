"""Row a7: unrestarted GMRES (oracle, fp64, modified Gram-Schmidt).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper solves every system with "a tolerance of 1e-6 and a maximum of 200
iterations" and names no method; reading R-gmres:
GMRES (Saad & Schultz 1986), x0 = 0, beta = ||b||_2, inner product <u,v> = sum conj(u) v,
Arnoldi by modified Gram-Schmidt, Givens rotations on the Hessenberg matrix; stop at
the first j with |gamma_{j+1}| <= tol * beta or j = max_iter; x = V_j y; the reported
residual is the true ||b - A x|| / beta.  b = 0 returns x = 0 after 0 iterations.
Pinned by tests/test_oracle_gmres.py (numpy.linalg.solve on the same A, b; residual <=
tol; zero rhs; non-convergence flag).
"""
import numpy as np


def gmres(matvec, b, tol=1e-6, max_iter=200):
    """Returns (x, info) with info = dict(iters, converged, rel_residual)."""
    b = np.asarray(b, dtype=np.complex128)
    n = b.size
    beta = np.linalg.norm(b)
    if beta == 0.0:
        return np.zeros(n, np.complex128), dict(iters=0, converged=1, rel_residual=0.0)
    if not np.isfinite(beta):
        raise FloatingPointError("non-finite right-hand side")
    m = max_iter
    V = np.zeros((m + 1, n), np.complex128)
    H = np.zeros((m + 1, m), np.complex128)
    cs = np.zeros(m, np.complex128)
    sn = np.zeros(m, np.complex128)
    gam = np.zeros(m + 1, np.complex128)
    gam[0] = beta
    V[0] = b / beta
    j_done = 0
    converged = 0
    for j in range(m):
        w = np.asarray(matvec(V[j]), dtype=np.complex128)
        for i in range(j + 1):
            H[i, j] = np.vdot(V[i], w)
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        if not np.isfinite(H[j + 1, j]):
            raise FloatingPointError("non-finite Arnoldi norm")
        if H[j + 1, j] != 0:
            V[j + 1] = w / H[j + 1, j]
        for i in range(j):  # apply previous rotations
            hi, hi1 = H[i, j], H[i + 1, j]
            H[i, j] = np.conj(cs[i]) * hi + np.conj(sn[i]) * hi1
            H[i + 1, j] = -sn[i] * hi + cs[i] * hi1
        a, bb = H[j, j], H[j + 1, j]
        den = np.sqrt(abs(a) ** 2 + abs(bb) ** 2)
        cs[j], sn[j] = (a / den, bb / den) if den != 0 else (1.0, 0.0)
        H[j, j] = np.conj(cs[j]) * a + np.conj(sn[j]) * bb
        H[j + 1, j] = 0.0
        gam[j + 1] = -sn[j] * gam[j]
        gam[j] = np.conj(cs[j]) * gam[j]
        j_done = j + 1
        if abs(gam[j + 1]) <= tol * beta or H[j + 1, j] == 0 and abs(gam[j + 1]) == 0:
            converged = 1
            break
    k = j_done
    y = np.zeros(k, np.complex128)
    for i in range(k - 1, -1, -1):
        y[i] = (gam[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
    x = V[:k].T @ y
    res = np.linalg.norm(b - matvec(x)) / beta
    if not np.isfinite(res):
        raise FloatingPointError("non-finite residual")
    return x, dict(iters=k, converged=converged, rel_residual=float(res))
