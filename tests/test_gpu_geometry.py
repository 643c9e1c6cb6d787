"""Rows a1 (mesh preparation) and a12 (listener grid): CUDA path vs oracle."""
import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import requires_cuda, soa_to_aos, to_np
from oracle import geometry, listeners

pytestmark = [pytest.mark.gpu, requires_cuda]


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


@pytest.mark.parametrize("name", ["ico3", "bowl", "c4scene", "cube1"])
def test_mesh_prepare_bitwise(name):
    nat = _nat()
    m = {"ico3": lambda: I.icosphere(3), "bowl": lambda: I.bowl(64, 12, 2),
         "c4scene": lambda: I.c4_geometry(9)[0],
         "cube1": lambda: I.slab(1, 1, 1, 1, 1, 1)}[name]()
    ref = geometry.mesh_prepare(m.v, m.t)
    geo = nat.nat_mesh_prepare(nat.Mesh.from_numpy(m.v, m.t))
    for key in ("centroid", "normal"):
        assert np.array_equal(soa_to_aos(getattr(geo, key)), ref[key]), key
    for key in ("area", "diam"):
        assert np.array_equal(to_np(getattr(geo, key)), ref[key]), key
    assert np.array_equal(to_np(geo.area_cdf), ref["cdf"])       # sequential order
    assert geo.total_area == ref["total_area"]
    assert tuple(geo.center) == tuple(ref["center"])          # sequential sums, every op rounded
    assert geo.bound_radius == ref["bound_radius"]
    assert abs(geo.volume - ref["volume"]) <= 1e-12 * abs(ref["volume"])


def test_mesh_prepare_errors():
    nat = _nat()
    m = I.icosphere(1)
    with pytest.raises(nat.NatError, match="SINGULAR"):
        nat.nat_mesh_prepare(nat.Mesh.from_numpy(m.v, m.t[:, [0, 2, 1]]))
    t = m.t.copy()
    t[5] = [t[5, 0], t[5, 0], t[5, 1]]
    with pytest.raises(nat.NatError, match="zero-area triangle 5"):
        nat.nat_mesh_prepare(nat.Mesh.from_numpy(m.v, t))


@pytest.mark.parametrize("dims", [(4, 4, 4), (32, 32, 32), (7, 3, 5), (1, 1, 1)])
def test_listener_grid(dims):
    nat = _nat()
    c, R = (0.1, -0.2, 0.05), 0.37
    x = nat.nat_listener_grid(c, R, *dims)
    ref = listeners.shell_grid(np.array(c), R, *dims)
    np.testing.assert_allclose(soa_to_aos(x), ref, rtol=0, atol=4e-16 * 3 * R * 4)


@pytest.mark.parametrize("n,seed,stream", [(1, 0, 0), (1000, 20250606, 3), (262_147, 7, 1 << 33)])
def test_listener_random_shell(n, seed, stream):
    """Reading R-listen-rand: same Philox draws (tag 1) and formula as the oracle; only
    the libm / CUDA transcendentals (cbrt, sincos, sqrt) differ, by ulps."""
    nat = _nat()
    c, R = (0.1, -0.2, 0.05), 0.37
    x = nat.nat_listener_random_shell(c, R, n, seed=seed, stream_id=stream)
    ref = listeners.random_shell(np.array(c), R, n, seed=seed, stream_id=stream)
    np.testing.assert_allclose(soa_to_aos(x), ref, rtol=0, atol=1e-15 * 3 * R * 8)


def test_listener_random_shell_errors():
    nat = _nat()
    from paper_2506_06190_b200.nat import NatError
    for bad in (dict(n=0), dict(R=-1.0), dict(r_lo=0.0), dict(r_lo=2.0, r_hi=1.0)):
        kw = dict(center=(0, 0, 0), R=1.0, n=4)
        kw.update(bad)
        with pytest.raises(NatError):
            nat.nat_listener_random_shell(kw.pop("center"), kw.pop("R"), kw.pop("n"), **kw)
