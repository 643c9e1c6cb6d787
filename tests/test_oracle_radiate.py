"""Pins of oracle.radiate (row a11) with exact boundary data."""
import numpy as np

import nat_inputs as I
from oracle import analytic, geometry, radiate


def _sphere(level=4):
    m = I.icosphere(level)
    return m, geometry.mesh_prepare(m.v, m.t)


def test_pulsating_sphere_extinction_and_exterior():
    m, geo = _sphere()
    k = 1.0
    pb = analytic.pulsating_sphere(1.0, k)            # exact boundary Dirichlet data
    src = radiate.bem_sources(m.v, m.t, geo, np.full((1, m.n_tri), pb), np.ones((1, m.n_tri)))
    x = np.array([[0.0, 0, 0], [0.0, 0.0, 2.0], [1.5, 1.5, 0.0]])
    p = radiate.radiate(src, [k], x)[0]
    assert abs(p[0]) < 5e-3 * abs(pb)                 # extinction inside (exact: 0)
    pe = analytic.pulsating_sphere(np.linalg.norm(x[1:], axis=1), k)
    assert np.max(np.abs(p[1:] - pe) / np.abs(pe)) < 5e-3


def test_point_source_reproduction():
    m, geo = _sphere()
    xs, k = np.array([0.1, -0.2, 0.3]), 3.0
    c, n = geo["centroid"], geo["normal"]
    pt = analytic.point_source(c, xs, k)
    gt = analytic.point_source_dn(c, n, xs, k)
    src = radiate.bem_sources(m.v, m.t, geo, pt[None], gt[None])
    x = I.random_points_in_shell(50, 1.5, 3.0, seed=3)
    p = radiate.radiate(src, [k], x)[0]
    pe = analytic.point_source(x, xs, k)
    assert np.linalg.norm(p - pe) / np.linalg.norm(pe) < 1e-2


def test_far_field_decay_and_mode_batching():
    m, geo = _sphere(3)
    src = radiate.bem_sources(m.v, m.t, geo, np.full((2, m.n_tri), 0.3 + 0.1j),
                              np.ones((2, m.n_tri)))
    x = np.array([[0, 0, 50.0], [0, 0, 100.0]])
    p = radiate.radiate(src, [1.0, 2.0], x)
    ratio = np.abs(p[:, 1]) / np.abs(p[:, 0])
    assert np.all(np.abs(ratio - 0.5) < 0.01)
    single = radiate.radiate((src[0], src[1], src[2], src[3][1:], src[4][1:]), [2.0], x)
    np.testing.assert_array_equal(single[0], p[1])
