"""Rows a8 (sampling), a9 (MC right-hand side), a10 (MC operator) and the full MC
solve: CUDA path vs oracle.  Samples are compared bit for bit (same Philox stream)."""
import math

import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import rel_l2, requires_cuda, soa_to_aos, to_np
from oracle import geometry, kernel, mc, radiate

pytestmark = [pytest.mark.gpu, requires_cuda]

TOL = {"fp32": 1e-4, "fp64": 1e-10}


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


def _case(m):
    nat = _nat()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    return geometry.mesh_prepare(m.v, m.t), mesh, nat.nat_mesh_prepare(mesh)


@pytest.mark.parametrize("name,M,seed,sid", [("bowl", 4096, 20250606, 0), ("bowl", 1001, 7, 3),
                                              ("c4", 2048, 20250606, 9), ("ico3", 1, 1, 2**40 + 5)])
def test_sampling_bitwise(name, M, seed, sid):
    nat = _nat()
    m = {"bowl": lambda: I.bowl(64, 12, 2), "c4": lambda: I.c4_geometry(9)[0],
         "ico3": lambda: I.icosphere(3)}[name]()
    geo, mesh, gg = _case(m)
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, M, seed, sid)
    smp, stri = nat.nat_mc_sample(mesh, gg, M, seed, sid)
    s = to_np(smp)
    assert np.array_equal(to_np(stri), tri)
    assert np.array_equal(s[:3].T, y)
    assert np.array_equal(s[3:].T, n)


def _system_case(M, seed=5):
    m = I.icosphere(3)
    geo, mesh, gg = _case(m)
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, M, seed)
    return m, geo, mesh, gg, y, n, tri


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("n_sys,eps", [(1, 0.0), (3, 0.0), (6, 0.0), (3, 0.004), (1, 0.05)])
def test_mc_operator_and_rhs_parity(prec, n_sys, eps):
    """a9 / a10 against the oracle's dense Eq. SYS; eps = 0 lets the library derive the
    default disk radius, eps > 0 is a caller radius (readings R-eps / R-weight: the library
    forms w = (|Gamma| - pi eps^2) / (M - 1) itself; the larger radius widens the fp64
    close-pair band of the fp32 path)."""
    nat = _nat()
    M = 2333     # dense enough that random samples form close pairs (fp64 path)
    m, geo, mesh, gg, y, n, tri = _system_case(M)
    ks = list(np.linspace(0.5, 6.0, n_sys))
    g = I.random_complex((n_sys, M), 11)
    p = I.random_complex((n_sys, M), 12)
    smp = torch.from_numpy(np.ascontiguousarray(np.concatenate([y.T, n.T]))).cuda()
    b = to_np(nat.nat_mc_rhs(smp, ks, torch.from_numpy(g).cuda(), geo["total_area"], eps, prec))
    Ap = to_np(nat.nat_mc_apply(smp, ks, torch.from_numpy(p).cuda(), geo["total_area"], eps, prec))
    for s, k in enumerate(ks):
        A_ref, b_ref = mc.system(y, n, g[s], k, geo["total_area"], eps if eps > 0 else None)
        assert rel_l2(b[s], b_ref) <= TOL[prec]
        assert rel_l2(Ap[s], A_ref @ p[s]) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_surface_pressure_parity(prec):
    nat = _nat()
    m = I.bowl(32, 8, 2)
    geo, mesh, gg = _case(m)
    M, seed = 700, 3
    ks = [0.5, 2.0, 4.5]
    g_tri = I.neumann_harmonics(m, 3)
    y, n, tri, p_ref, infos = mc.surface_pressure(m.v, m.t, geo, ks, g_tri, M, seed, tol=1e-13)
    tol = 1e-6 if prec == "fp32" else 1e-12
    smp, stri, p, ginfo = nat.nat_mc_surface_pressure(mesh, gg, ks, torch.from_numpy(g_tri).cuda(), M, seed,
                                                      prec=prec, tol=tol)
    assert np.array_equal(to_np(stri), tri)
    for s in range(3):
        # the true residual of the fp32 path is floored by the fp32 operator (~1e-7)
        assert ginfo[s]["converged"] == 1 and ginfo[s]["rel_residual"] <= (1e-5 if prec == "fp32" else 2 * tol)
        assert rel_l2(to_np(p)[s], p_ref[s]) <= TOL[prec]
    # radiated field of the MC solution (MC sources, w = |Gamma|/M)
    src = nat.nat_mc_sources(smp, gg.total_area, p, torch.from_numpy(g_tri[:, tri]).cuda(), center=gg.center)
    x = I.random_points_in_shell(300, 1.6, 3.0, seed=2) + np.asarray(geo["center"])
    out = to_np(nat.nat_radiate_field(src, ks, torch.from_numpy(np.ascontiguousarray(x.T)).cuda(), prec=prec))
    ref = radiate.radiate(radiate.mc_sources(y, n, geo["total_area"], p_ref, g_tri[:, tri]), ks, x)
    for s in range(3):
        assert rel_l2(out[s], ref[s]) <= TOL[prec]


def test_degenerate_cases():
    nat = _nat()
    m = I.icosphere(2)
    geo, mesh, gg = _case(m)
    g = torch.from_numpy(np.full((1, m.n_tri), 2.0 + 1.0j)).cuda()
    # M = 1: 1/2 p = -(eps/2) g  ->  p = -eps g  (reading R-sign); the fp32 solve keeps its
    # Krylov basis in fp32 (reading R-basis32), so it is exact to fp32 rounding only
    eps = math.sqrt(gg.total_area / math.pi)
    for prec, tol in (("fp64", 1e-12), ("fp32", 1e-7)):
        smp, stri, p, info = nat.nat_mc_surface_pressure(mesh, gg, [1.0], g, 1, seed=4, prec=prec)
        assert abs(to_np(p)[0, 0] - (-eps * (2.0 + 1.0j))) <= tol * abs(eps * (2.0 + 1.0j))
    # g = 0 -> p = 0 after 0 iterations
    _, _, p0, i0 = nat.nat_mc_surface_pressure(mesh, gg, [1.0, 3.0], torch.zeros(2, m.n_tri, dtype=torch.complex128,
                                                                                 device="cuda"), 256, seed=4)
    assert torch.count_nonzero(p0) == 0 and i0[0]["iters"] == 0
    # coincident samples -> NAT_ERR_SINGULAR naming the pair
    smp, stri = nat.nat_mc_sample(mesh, gg, 50, 1)
    smp[:, 17] = smp[:, 4]
    stri[17] = stri[4]
    with pytest.raises(nat.NatError, match=r"coincident samples \(4, 17\)"):
        nat.nat_mc_surface_pressure(mesh, gg, [1.0], g, 50, samples_in=smp, sample_tri_in=stri)


def test_c3_launch_configuration():
    """Config C3: bowl 49,664 tri, M = 4096 uniform samples, 32 modes k_m a = 0.5 +
    7.5 m / 31, fp32, tol 1e-6: the GPU solution satisfies sampled rows of the oracle's
    system (property that holds at any size) and samples are bitwise identical."""
    nat = _nat()
    m = I.bowl()
    geo, mesh, gg = _case(m)
    M = 4096
    ks = I.c3_wavenumbers()
    g_tri = I.neumann_harmonics(m, 32)
    smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, gg, ks, torch.from_numpy(g_tri).cuda(), M,
                                                      seed=I.SEED, stream_id=0)
    assert all(i["converged"] == 1 for i in infos)
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, M, I.SEED, 0)
    assert np.array_equal(to_np(stri), tri)
    P = to_np(p)
    eps, w = mc.default_eps(geo["total_area"], M), None
    w = mc.weight(geo["total_area"], M, eps)
    rows = np.random.default_rng(1).choice(M, 16, replace=False)
    for s in (0, 13, 31):
        k = ks[s]
        g = g_tri[s][tri]
        res, nb = [], []
        for i in rows:
            j = np.arange(M) != i
            Ai = -w * kernel.green_dn_y(y[i], y[j], n[j], k)
            bi = -w * np.sum(kernel.green(y[i], y[j], k) * g[j]) - 0.5 * eps * g[i]
            res.append(0.5 * P[s, i] + Ai @ P[s, j] - bi)
            nb.append(bi)
        assert np.linalg.norm(res) / np.linalg.norm(nb) <= 1e-4


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_mc_operator_row_blocks_ragged(prec):
    """SURVEY §8(e) row sharding of the MC operator: rows [r0, r1) of three ragged blocks
    (as ranks 0..2 of 3 own them) against the oracle's operator rows."""
    nat = _nat()
    M = 2333
    m, geo, mesh, gg, y, n, tri = _system_case(M)
    ks = [0.5, 3.0, 6.0]
    area, eps = geo["total_area"], 0.0
    p = I.random_complex((3, M), 21)
    smp = torch.from_numpy(np.ascontiguousarray(np.concatenate([y.T, n.T]))).cuda()
    pt = torch.from_numpy(p).cuda()
    full = to_np(nat.nat_mc_apply(smp, ks, pt, area, eps, prec))
    blocks = []
    for r in range(3):
        r0, r1 = nat.row_range(M, r, 3)
        blocks.append(to_np(nat.nat_mc_apply_rows(smp, ks, pt, area, eps, r0, r1, prec)))
    got = np.concatenate(blocks, axis=1)
    for s, k in enumerate(ks):
        A_ref, _ = mc.system(y, n, np.zeros(M), k, geo["total_area"])
        assert rel_l2(got[s], A_ref @ p[s]) <= TOL[prec]
    assert rel_l2(got, full) <= (1e-6 if prec == "fp32" else 1e-13)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_sharded_surface_pressure_world1_matches(prec):
    """The row-sharded solve on one rank (comm = NULL) reproduces the batched solve and the
    oracle (same samples, same iterations)."""
    nat = _nat()
    m = I.bowl(32, 8, 2)
    geo, mesh, gg = _case(m)
    M, seed = 700, 3
    ks = [0.5, 2.0, 4.5]
    g_tri = I.neumann_harmonics(m, 3)
    y, n, tri, p_ref, infos = mc.surface_pressure(m.v, m.t, geo, ks, g_tri, M, seed, tol=1e-13)
    tol = 1e-6 if prec == "fp32" else 1e-12
    gt = torch.from_numpy(g_tri).cuda()
    smp, stri, p, info = nat.nat_mc_surface_pressure_sharded(mesh, gg, ks, gt, M, None, seed, prec=prec, tol=tol)
    _, _, p0, info0 = nat.nat_mc_surface_pressure(mesh, gg, ks, gt, M, seed, prec=prec, tol=tol)
    assert np.array_equal(to_np(stri), tri)
    for s in range(3):
        assert info[s]["converged"] == 1
        assert abs(info[s]["iters"] - info0[s]["iters"]) <= 1
        assert rel_l2(to_np(p)[s], p_ref[s]) <= TOL[prec]
        assert rel_l2(to_np(p)[s], to_np(p0)[s]) <= (1e-5 if prec == "fp32" else 1e-11)


def test_row_api_errors():
    nat = _nat()
    M = 300
    m, geo, mesh, gg, y, n, tri = _system_case(M)
    area = geo["total_area"]
    smp = torch.from_numpy(np.ascontiguousarray(np.concatenate([y.T, n.T]))).cuda()
    p = torch.ones(1, M, dtype=torch.complex128, device="cuda")
    for r0, r1 in ((0, 0), (5, 3), (0, M + 1), (-1, 10)):
        with pytest.raises(nat.NatError, match="row range"):
            nat.nat_mc_apply_rows(smp, [1.0], p, area, 0.0, r0, r1)
    with pytest.raises(nat.NatError):
        nat.nat_mc_apply_rows(smp, [1.0], p.cpu(), area, 0.0, 0, 10)     # host tensor
    with pytest.raises(nat.NatError, match="total_area"):
        nat.nat_mc_apply(smp, [1.0], p, -1.0)
    with pytest.raises(nat.NatError, match="disk area"):
        nat.nat_mc_apply(smp, [1.0], p, area, 10.0)                       # pi eps^2 > |Gamma|
    with pytest.raises(nat.NatError, match="M must be"):
        nat.nat_mc_surface_pressure_sharded(mesh, gg, [1.0], torch.ones(1, m.n_tri, dtype=torch.complex128,
                                                                         device="cuda"), 1)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_surface_pressure_caller_eps(prec):
    """The whole solve at a caller disk radius (opts->eps > 0; readings R-eps, R-weight:
    the library forms w = (|Gamma| - pi eps^2)/(M - 1)) against the oracle at the same eps."""
    nat = _nat()
    m = I.bowl(32, 8, 2)
    geo, mesh, gg = _case(m)
    M, seed, eps = 500, 5, 0.03
    ks = [1.0, 3.0]
    g_tri = I.neumann_harmonics(m, 2)
    y, n, tri, p_ref, _ = mc.surface_pressure(m.v, m.t, geo, ks, g_tri, M, seed, eps=eps, tol=1e-13)
    _, _, _, p_def, _ = mc.surface_pressure(m.v, m.t, geo, ks, g_tri, M, seed, tol=1e-13)
    tol = 1e-6 if prec == "fp32" else 1e-12
    _, _, p, info = nat.nat_mc_surface_pressure(mesh, gg, ks, torch.from_numpy(g_tri).cuda(), M, seed, eps=eps,
                                                prec=prec, tol=tol)
    for s in range(2):
        assert info[s]["converged"] == 1
        assert rel_l2(to_np(p)[s], p_ref[s]) <= TOL[prec]
        assert rel_l2(p_def[s], p_ref[s]) > 100 * TOL[prec]   # the radius changes the solution


def test_solve_groups_agree():
    """nat_mc_set_groups: the batch split into 1, 2 or 4 concurrently iterating groups
    gives the same solution (same arithmetic per system; launch shapes may change the
    rounding) and the same iteration counts within one."""
    nat = _nat()
    m = I.bowl(32, 8, 2)
    geo, mesh, gg = _case(m)
    M, seed = 700, 3
    ks = list(np.linspace(0.5, 6.0, 7))
    g_tri = torch.from_numpy(I.neumann_harmonics(m, 7)).cuda()
    out = {}
    try:
        for G in (1, 2, 4):
            nat.nat_mc_set_groups(G)
            _, _, p, info = nat.nat_mc_surface_pressure(mesh, gg, ks, g_tri, M, seed, prec="fp32", tol=1e-6)
            out[G] = (to_np(p), [i["iters"] for i in info], [i["converged"] for i in info])
    finally:
        nat.nat_mc_set_groups(1)
    for G in (2, 4):
        assert rel_l2(out[G][0], out[1][0]) <= 1e-6
        assert all(abs(a - b) <= 1 for a, b in zip(out[G][1], out[1][1]))
        assert all(out[G][2])
    with pytest.raises(nat.NatError):
        nat.nat_mc_set_groups(5)


def test_krylov_config_shapes_agree():
    """nat_krylov_config: the fused Arnoldi step with 2 / 4 / 8 CTAs per system and 256 /
    512 threads gives the same solution (summation order only) and iteration counts within
    one; invalid shapes are rejected."""
    nat = _nat()
    m = I.bowl(32, 8, 2)
    geo, mesh, gg = _case(m)
    M, seed = 700, 3
    ks = list(np.linspace(0.5, 6.0, 5))
    g_tri = torch.from_numpy(I.neumann_harmonics(m, 5)).cuda()
    out = {}
    try:
        for cfg in ((4, 512, 120), (2, 256, 0), (2, 512, 0), (4, 256, 0), (8, 512, 120)):
            nat.nat_krylov_config(*cfg)
            _, _, p, info = nat.nat_mc_surface_pressure(mesh, gg, ks, g_tri, M, seed, prec="fp32", tol=1e-6)
            out[cfg] = (to_np(p), [i["iters"] for i in info])
    finally:
        nat.nat_krylov_config(4, 512, 120)
    ref = out[(4, 512, 120)]
    for cfg, (p, it) in out.items():
        assert rel_l2(p, ref[0]) <= 1e-6, cfg
        assert all(abs(a - b) <= 1 for a, b in zip(it, ref[1])), cfg
    for bad in ((3, 512, 120), (4, 128, 120), (4, 512, -1)):
        with pytest.raises(nat.NatError):
            nat.nat_krylov_config(*bad)
