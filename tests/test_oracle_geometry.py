"""Pins of oracle.geometry (row a1)."""
import math

import numpy as np
import pytest

import nat_inputs as I
from oracle import geometry


def test_hand_triangle_in_tetrahedron():
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 2, 0], [0, 0, 3]], dtype=float)
    t = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]])
    g = geometry.mesh_prepare(v, t)
    assert g["area"][0] == 1.0
    np.testing.assert_array_equal(g["normal"][0], [0, 0, -1])
    np.testing.assert_allclose(g["centroid"][0], [1 / 3, 2 / 3, 0], rtol=0, atol=1e-16)
    assert g["diam"][0] == math.sqrt(5)
    assert abs(g["volume"] - 1.0) < 1e-15          # 1*2*3/6
    np.testing.assert_allclose((g["area"][:, None] * g["normal"]).sum(0), 0, atol=1e-15)
    assert g["cdf"][-1] == g["total_area"]


def test_sphere_convergence():
    errs = []
    for L in (2, 3, 4):
        m = I.icosphere(L)
        g = geometry.mesh_prepare(m.v, m.t)
        errs.append(abs(g["total_area"] - 4 * math.pi) / (4 * math.pi))
        np.testing.assert_allclose((g["area"][:, None] * g["normal"]).sum(0), 0, atol=1e-13)
        assert abs(g["bound_radius"] - 1) < 1e-12
        assert np.all(np.diff(g["cdf"]) > 0)
    assert errs[0] / errs[1] > 3.5 and errs[1] / errs[2] > 3.5   # O(h^2)
    assert errs[2] < 2e-3


def test_rejects_inward_and_degenerate():
    m = I.icosphere(1)
    with pytest.raises(ValueError):
        geometry.mesh_prepare(m.v, m.t[:, [0, 2, 1]])
    t = m.t.copy()
    t[3] = [t[3, 0], t[3, 0], t[3, 1]]
    with pytest.raises(ValueError):
        geometry.mesh_prepare(m.v, t)


def test_bowl_volume_and_centre():
    m = I.bowl(128, 24, 2)
    g = geometry.mesh_prepare(m.v, m.t)
    exact = 2 / 3 * math.pi * (1 - 0.9 ** 3)
    assert abs(g["volume"] - exact) / exact < 5e-3
    assert abs(g["center"][0]) < 1e-12 and abs(g["center"][1]) < 1e-12


def test_centre_is_the_area_weighted_surface_centroid():
    """centre = sum A_t c_t / |Gamma| (R-geom): a box's centre is its centre (exact up to
    rounding) and R its half diagonal; the thick bowl's centre converges O(h^2) to the
    analytic surface centroid z = (2 pi (-1/2) + 2 pi 0.81 (-0.45)) / (3.81 pi) (outer and
    inner hemispherical surfaces, rim annulus at z = 0)."""
    m = I.slab(0.4, 0.3, 0.2, 4, 3, 2, centre=(0.1, -0.2, 0.3))
    g = geometry.mesh_prepare(m.v, m.t)
    np.testing.assert_allclose(g["center"], [0.1, -0.2, 0.3], rtol=0, atol=2e-16)
    assert abs(g["bound_radius"] - math.sqrt(0.2 ** 2 + 0.15 ** 2 + 0.1 ** 2)) < 2e-16
    exact = -1.729 / 3.81
    errs = []
    for n_az, n_psi in ((32, 8), (64, 16), (128, 32)):
        z = geometry.mesh_prepare(*(lambda b: (b.v, b.t))(I.bowl(n_az, n_psi, 2)))["center"][2]
        errs.append(abs(z - exact))
    assert errs[0] / errs[1] > 3.5 and errs[1] / errs[2] > 3.5 and errs[2] < 2e-4
