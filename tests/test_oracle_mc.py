"""Pins of oracle.mc (rows a8-a10): sampler properties, degenerate systems, and the
pulsating-sphere statistics (the MC realisation itself is parity-unpinned pointwise)."""
import math

import numpy as np
import pytest
from scipy import stats

import nat_inputs as I
from oracle import analytic, geometry, listeners, mc, radiate


def test_samples_on_their_triangles_with_triangle_normals():
    m = I.bowl(32, 8, 2)
    geo = geometry.mesh_prepare(m.v, m.t)
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, 5000, seed=7, stream_id=3)
    v1, v2, v3 = (m.v[m.t[tri, a]] for a in range(3))
    # barycentric residual: solve y = v1 + s(v2-v1) + t(v3-v1) in the plane
    e1, e2, d = v2 - v1, v3 - v1, y - v1
    G = np.stack([np.einsum("ij,ij->i", e1, e1), np.einsum("ij,ij->i", e1, e2),
                  np.einsum("ij,ij->i", e2, e2)], 1)
    r1, r2 = np.einsum("ij,ij->i", d, e1), np.einsum("ij,ij->i", d, e2)
    det = G[:, 0] * G[:, 2] - G[:, 1] ** 2
    s = (G[:, 2] * r1 - G[:, 1] * r2) / det
    t = (G[:, 0] * r2 - G[:, 1] * r1) / det
    res = np.linalg.norm(v1 + s[:, None] * e1 + t[:, None] * e2 - y, axis=1)
    assert np.max(res) < 1e-12
    assert np.all(s >= -1e-12) and np.all(t >= -1e-12) and np.all(s + t <= 1 + 1e-12)
    np.testing.assert_array_equal(n, geo["normal"][tri])


def test_face_frequencies_chi2_on_cube():
    m = I.slab(1, 1, 1, 3, 3, 3)     # unit cube, 6 faces of equal area
    geo = geometry.mesh_prepare(m.v, m.t)
    M = 60000
    y, _, _ = mc.sample_uniform(m.v, m.t, geo, M, seed=11)
    face = np.argmax(np.abs(y) * 2 > 1 - 1e-12, axis=1) * 2 + (y[np.arange(M), np.argmax(np.abs(y) * 2 > 1 - 1e-12, axis=1)] > 0)
    counts = np.bincount(face, minlength=6)
    assert counts.sum() == M
    assert stats.chisquare(counts).pvalue > 1e-3
    # and uniform within a face: x-coordinate of +z face hits is U(-1/2,1/2)
    top = y[np.abs(y[:, 2] - 0.5) < 1e-12]
    assert stats.kstest(top[:, 0] + 0.5, "uniform").pvalue > 1e-3


def test_default_eps_gives_weight_area_over_M():
    for M in (10, 1000, 4096):
        eps = mc.default_eps(4 * math.pi, M)
        assert abs(mc.weight(4 * math.pi, M, eps) - 4 * math.pi / M) < 1e-14


def test_single_sample_row():
    # M = 1: 1/2 p = -(eps/2) g  =>  p = -eps g   (disk term only, reading R-sign)
    y = np.array([[0.0, 0.0, 1.0]])
    n = np.array([[0.0, 0.0, 1.0]])
    A, b = mc.system(y, n, np.array([2.0 + 1j]), 1.0, 4 * math.pi)
    eps = math.sqrt(4 * math.pi / math.pi)
    assert A[0, 0] == 0.5
    assert abs(b[0] / A[0, 0] - (-eps * (2.0 + 1j))) < 1e-15


def test_zero_neumann_gives_zero_pressure():
    m = I.icosphere(2)
    geo = geometry.mesh_prepare(m.v, m.t)
    _, _, _, p, infos = mc.surface_pressure(m.v, m.t, geo, [1.0], np.zeros((1, m.n_tri)), 200, 1)
    assert np.all(p == 0) and infos[0]["iters"] == 0


def test_coincident_samples_raise():
    y = np.array([[0.0, 0, 1], [0.3, 0, 0.9], [0.0, 0, 1]])
    n = y / np.linalg.norm(y, axis=1, keepdims=True)
    with pytest.raises(ZeroDivisionError):
        mc.system(y, n, np.ones(3), 1.0, 4 * math.pi)


def test_pulsating_sphere_statistics():
    """Seed-averaged MC solution approaches the analytic pulsating sphere: exterior
    field within 5% per seed-average, boundary mean within the O(eps) disk bias + noise
    (the dropped disk dG term biases the diagonal by eps/4)."""
    m = I.icosphere(4)
    geo = geometry.mesh_prepare(m.v, m.t)
    g = I.neumann_constant(m)
    k, M = 1.0, 1000
    L = listeners.shell_grid(np.zeros(3), 1.0, 4, 4, 2)
    pe = analytic.pulsating_sphere(np.linalg.norm(L, axis=1), k)
    fields, means = [], []
    for seed in range(4):
        y, n, tri, p, infos = mc.surface_pressure(m.v, m.t, geo, [k], g[None], M, seed)
        assert infos[0]["converged"] == 1 and infos[0]["rel_residual"] < 1e-6
        src = radiate.mc_sources(y, n, geo["total_area"], p, g[tri][None])
        fields.append(radiate.radiate(src, [k], L)[0])
        means.append(np.mean(p[0]))
    f = np.mean(fields, axis=0)
    assert np.linalg.norm(f - pe) / np.linalg.norm(pe) < 0.05
    pb = analytic.pulsating_sphere(1.0, k)
    assert abs(np.mean(means) - pb) / abs(pb) < 0.10


@pytest.mark.parametrize("M", [2, 5, 10])
def test_weight_at_a_caller_eps_conserves_the_sampling_surface(M):
    """Reading R-weight ("reduction in the sampling surface corresponding to the area
    of the small disk"): the M - 1 off-disk weights and the disk area add up to |Gamma| for
    any caller eps, and only the default eps gives |Gamma| / M."""
    area = 3.7
    for eps in (1e-3, 0.05, 0.3, mc.default_eps(area, M)):
        w = mc.weight(area, M, eps)
        assert abs(w * (M - 1) + math.pi * eps * eps - area) < 1e-14 * area
    assert abs(mc.weight(area, M, 0.3) - area / M) > 1e-3


@pytest.mark.parametrize("M,k,eps", [(3, 0.0, None), (7, 2.5, 0.11), (10, 6.0, 0.02)])
def test_small_system_entries_brute_force(M, k, eps):
    """M <= 10 hand systems: every entry against properties that do not reuse
    the oracle's kernel formulas — A_ij (i != j) is -w times the central finite difference of
    G(y_i, .) along n_j at y_j (pins the derivative, its sign and which normal enters);
    with g = e_j, b_i = -w G(y_i, y_j) has modulus w / (4 pi r_ij) and phase k r_ij + pi,
    and b_j = -(eps/2) (the disk term at the caller's eps); A_ii = 1/2."""
    rng = np.random.default_rng(M)
    d = rng.normal(size=(M, 3))
    y = d / np.linalg.norm(d, axis=1, keepdims=True)
    n = y.copy()
    area = 4 * math.pi
    e = mc.default_eps(area, M) if eps is None else eps
    w = mc.weight(area, M, e)
    for j in range(M):
        g = np.zeros(M)
        g[j] = 1.0
        A, b = mc.system(y, n, g, k, area, eps)
        assert A[j, j] == 0.5
        assert abs(b[j] - (-0.5 * e)) < 1e-15
        for i in range(M):
            if i == j:
                continue
            h = 1e-5
            gp = np.exp(1j * k * np.linalg.norm(y[j] + h * n[j] - y[i])) / (4 * math.pi * np.linalg.norm(y[j] + h * n[j] - y[i]))
            gm = np.exp(1j * k * np.linalg.norm(y[j] - h * n[j] - y[i])) / (4 * math.pi * np.linalg.norm(y[j] - h * n[j] - y[i]))
            fd = (gp - gm) / (2 * h)
            assert abs(A[i, j] - (-w * fd)) < 1e-6 * max(1.0, abs(w * fd))   # O(h^2) FD error
            r = np.linalg.norm(y[i] - y[j])
            assert abs(abs(b[i]) - w / (4 * math.pi * r)) < 1e-14
            if k > 0:
                ph = (np.angle(b[i]) - (k * r + math.pi)) % (2 * math.pi)
                assert min(ph, 2 * math.pi - ph) < 1e-12
