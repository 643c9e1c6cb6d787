"""NEXT-3: Poisson-disk boundary samples on the GPU vs oracle/poisson.py (bit for bit, the
same accepted candidate indices), the blue-noise properties at the C3 size, and the MC
solve fed with Poisson samples (reading R-poisson)."""
import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import rel_l2, requires_cuda, soa_to_aos, to_np
from oracle import geometry, mc, poisson

pytestmark = [pytest.mark.gpu, requires_cuda]


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


def _case(m):
    nat = _nat()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    return geometry.mesh_prepare(m.v, m.t), mesh, nat.nat_mesh_prepare(mesh)


@pytest.mark.parametrize("name,M,seed,sid", [("ico3", 300, 11, 2), ("bowl", 600, 20250606, 0),
                                              ("cube", 150, 5, 2**33 + 1)])
def test_poisson_bitwise(name, M, seed, sid):
    nat = _nat()
    m = {"ico3": lambda: I.icosphere(3), "bowl": lambda: I.bowl(48, 12, 2), "cube": lambda: I.cubed_sphere(4)}[name]()
    geo, mesh, gg = _case(m)
    smp, stri, r = nat.nat_mc_poisson_sample(mesh, gg, M, seed=seed, stream_id=sid)
    # the oracle uses its own a1 frame (centre and radius are bit-identical, test_gpu_geometry)
    y, n, tri, cand, r_o = poisson.sample(m.v, m.t, geo, M, seed, sid)
    assert r == r_o
    assert np.array_equal(to_np(stri), tri)
    x = soa_to_aos(smp[:3])
    assert np.array_equal(x, y) and np.array_equal(soa_to_aos(smp[3:]), n)


def test_poisson_c3_properties():
    """C3 size (bowl, M_target = 4096): minimum distance >= r (all pairs) and every
    candidate of the pool within r of a sample (maximality), computed with torch."""
    nat = _nat()
    m = I.bowl()
    geo, mesh, gg = _case(m)
    M = 4096
    smp, stri, r = nat.nat_mc_poisson_sample(mesh, gg, M, seed=20250606)
    y = smp[:3].T.contiguous()
    k = y.shape[0]
    assert 0.8 * M <= k <= 1.6 * M
    d2 = torch.cdist(y, y).pow(2)
    d2.fill_diagonal_(float("inf"))
    assert d2.min().item() >= r * r * (1 - 1e-12)
    # the candidate pool = the a8 sampler with tag 2 (oracle check on a prefix)
    yc, _, _ = mc.sample_uniform(m.v, m.t, geo, 1000, 20250606, 0, tag=2)
    pool = torch.from_numpy(mc.sample_uniform(m.v, m.t, geo, 30 * M, 20250606, 0, tag=2)[0]).cuda()
    assert np.array_equal(pool[:1000].cpu().numpy(), yc)
    dmin = torch.cat([torch.cdist(pool[i:i + 8192], y).min(dim=1).values for i in range(0, pool.shape[0], 8192)])
    assert dmin.max().item() < r * (1 + 1e-12)


def test_mc_solve_with_poisson_samples():
    """nat_mc_surface_pressure fed with GPU Poisson samples (opts->samples_in) vs the oracle
    system on the same samples."""
    nat = _nat()
    m = I.bowl(32, 8, 2)
    geo, mesh, gg = _case(m)
    smp, stri, r = nat.nat_mc_poisson_sample(mesh, gg, 500, seed=9)
    M = smp.shape[1]
    ks = [0.5, 3.0]
    g_tri = I.neumann_harmonics(m, 2)
    y = soa_to_aos(smp[:3])
    tri = to_np(stri)
    _, _, _, p_ref, _ = mc.surface_pressure(m.v, m.t, geo, ks, g_tri, M, 0, tol=1e-13,
                                            samples=(y, soa_to_aos(smp[3:]), tri))
    _, _, p, info = nat.nat_mc_surface_pressure(mesh, gg, ks, torch.from_numpy(g_tri).cuda(), M, 0, prec="fp32",
                                                tol=1e-6, samples_in=smp.contiguous(), sample_tri_in=stri)
    for s in range(2):
        assert info[s]["converged"] == 1
        assert rel_l2(to_np(p)[s], p_ref[s]) <= 1e-4


def test_poisson_errors():
    nat = _nat()
    from paper_2506_06190_b200.nat import NatError
    m = I.icosphere(2)
    _, mesh, gg = _case(m)
    with pytest.raises(NatError):
        nat.nat_mc_poisson_sample(mesh, gg, 0)
    with pytest.raises(NatError):   # grid finer than 1280^3 cells
        nat.nat_mc_poisson_sample(mesh, gg, 10, r=1e-4)
