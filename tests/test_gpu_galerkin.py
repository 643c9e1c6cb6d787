"""NEXT-2: Galerkin P0 assembly (nat_quad_opts.galerkin, reading
R-galerkin) on the GPU against oracle/galerkin.py — whole operators on a small sphere,
sampled rows on the bowl (sharp rim edges) and at the C2 size, ragged row blocks, the
solve against the oracle's solution and the analytic pulsating / oscillating sphere."""
import functools

import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import rel_l2, requires_cuda, soa_to_aos, to_np
from oracle import analytic, galerkin, geometry, nearlist

pytestmark = [pytest.mark.gpu, requires_cuda]

TOL = {"fp32": 1e-4, "fp64": 1e-10}


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


@functools.lru_cache(maxsize=None)
def _oracle_full(level, k):
    m = I.icosphere(level)
    geo = geometry.mesh_prepare(m.v, m.t)
    near = nearlist.near_list(m.t, geo["centroid"], geo["diam"])
    g = I.neumann_rigid_z(m)
    A, b = galerkin.assemble(m.v, m.t, geo, k, g[None], near=near)
    return m, g, A, b


def _gpu(m, g, k, prec, r0=0, r1=None, ss_order=0):
    nat = _nat()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    o = nat.quad_opts(galerkin=True, ss_order=ss_order)
    nl = nat.nat_bem_near_list(mesh, gg, r0, r1 or m.n_tri, opts=o)
    A, b = nat.nat_bem_assemble(mesh, gg, nl, k, torch.from_numpy(g[None]).cuda(), prec=prec, opts=o)
    return mesh, gg, A, b


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("k", [1.0, 4.0])
def test_galerkin_whole_operator(prec, k):
    m, g, A_r, b_r = _oracle_full(2, k)
    _, _, A, b = _gpu(m, g, k, prec)
    A_g = to_np(A)[:, : m.n_tri].astype(np.complex128)
    assert rel_l2(A_g, A_r) <= TOL[prec]
    assert rel_l2(to_np(b[0]), b_r[0]) <= TOL[prec]
    # the diagonal is exactly |T_i| / 2 (K_ii = 0 on a flat triangle)
    geo = geometry.mesh_prepare(m.v, m.t)
    assert np.allclose(np.diag(A_g).real, 0.5 * geo["area"], rtol=1e-6 if prec == "fp32" else 1e-15)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_galerkin_ragged_row_blocks_and_ss_order(prec):
    k = 2.0
    m = I.icosphere(3)
    g = I.neumann_rigid_z(m)
    geo = geometry.mesh_prepare(m.v, m.t)
    for r0, r1, n in ((0, 427, 4), (427, 854, 4), (854, 1280, 6)):
        _, _, A, b = _gpu(m, g, k, prec, r0, r1, ss_order=n)
        rows = np.array([r0, (r0 + r1) // 2, r1 - 1])
        A_ref, b_ref = galerkin.assemble(m.v, m.t, geo, k, g[None], rows=rows, opts=dict(ss_order=n))
        A_g = to_np(A)[rows - r0, : m.n_tri].astype(np.complex128)
        assert rel_l2(A_g, A_ref) <= TOL[prec]
        assert rel_l2(to_np(b[0])[rows - r0], b_ref[0]) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_galerkin_bowl_sampled_rows(prec):
    """The thick bowl: rim edges with 90-degree dihedral angles (edge/vertex pairs that
    are far from coplanar) and the thin wall (close pairs across it)."""
    m = I.bowl(32, 8, 2)
    g = I.neumann_harmonics(m, 3)[2].astype(np.complex128)
    k = 3.0
    geo = geometry.mesh_prepare(m.v, m.t)
    _, _, A, b = _gpu(m, g, k, prec)
    rows = np.random.default_rng(7).choice(m.n_tri, 6, replace=False)
    # rim rows: centroid near z = 0
    rim = np.argsort(np.abs(geo["centroid"][:, 2]))[:3]
    rows = np.concatenate([rows, rim])
    A_ref, b_ref = galerkin.assemble(m.v, m.t, geo, k, g[None], rows=rows)
    A_g = to_np(A)[rows, : m.n_tri].astype(np.complex128)
    assert rel_l2(A_g, A_ref) <= TOL[prec]
    assert rel_l2(to_np(b[0])[rows], b_ref[0]) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_galerkin_solve_matches_oracle(prec):
    nat = _nat()
    k = 1.0
    m, g, A_r, b_r = _oracle_full(2, k)
    _, _, A, b = _gpu(m, g, k, prec)
    tol = 1e-6 if prec == "fp32" else 1e-12
    x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=tol)
    assert info["converged"] == 1
    assert rel_l2(to_np(x), np.linalg.solve(A_r, b_r[0])) <= TOL[prec]


def test_galerkin_analytic_spheres():
    """Galerkin assembly + GMRES + radiation on the GPU (fp32): pulsating sphere at k = 1
    (C1 mesh) and the oscillating sphere at ka = 2 and 8 (icosphere L4) within 2 %."""
    nat = _nat()
    m3 = I.icosphere(3)
    mesh, gg, A, b = _gpu(m3, I.neumann_constant(m3), 1.0, "fp32")
    x, info = nat.nat_bem_solve(A, b[0], m3.n_tri, tol=1e-6)
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 4, 4, 4)
    gt = torch.from_numpy(I.neumann_constant(m3)[None]).cuda()
    p = to_np(nat.nat_radiate_field(nat.nat_bem_sources(mesh, gg, x[None], gt), [1.0], lis))[0]
    pe = analytic.pulsating_sphere(np.linalg.norm(soa_to_aos(lis), axis=1), 1.0)
    assert rel_l2(p, pe) <= 0.02
    m4 = I.icosphere(4)
    g4 = I.neumann_rigid_z(m4)
    for ka in (2.0, 8.0):
        mesh, gg, A, b = _gpu(m4, g4, ka, "fp32")
        x, info = nat.nat_bem_solve(A, b[0], m4.n_tri, tol=1e-6)
        lis = nat.nat_listener_grid((0, 0, 0), 1.0, 8, 8, 2)
        src = nat.nat_bem_sources(mesh, gg, x[None], torch.from_numpy(g4[None]).cuda())
        p = to_np(nat.nat_radiate_field(src, [ka], lis))[0]
        assert rel_l2(p, analytic.oscillating_sphere(soa_to_aos(lis), ka)) <= 0.02


def test_c2_galerkin_fp32_sampled_rows():
    """C2 size (icosphere L5, 20,480 tri, ka = 8): sampled rows of the Galerkin operator."""
    m = I.icosphere(5)
    g = I.neumann_rigid_z(m)
    ka = 8.0
    _, _, A, b = _gpu(m, g, ka, "fp32")
    geo = geometry.mesh_prepare(m.v, m.t)
    rows = np.random.default_rng(3).choice(m.n_tri, 4, replace=False)
    A_ref, b_ref = galerkin.assemble(m.v, m.t, geo, ka, g[None], rows=rows)
    A_g = to_np(A[torch.from_numpy(rows).cuda()])[:, : m.n_tri].astype(np.complex128)
    assert rel_l2(A_g, A_ref) <= 1e-4
    assert rel_l2(to_np(b[0])[rows], b_ref[0]) <= 1e-4


def test_galerkin_rejects_burton_miller():
    nat = _nat()
    m = I.icosphere(1)
    with pytest.raises(nat.NatError, match="Galerkin"):
        mesh = nat.Mesh.from_numpy(m.v, m.t)
        gg = nat.nat_mesh_prepare(mesh)
        o = nat.quad_opts(galerkin=True, burton_miller=True)
        nl = nat.nat_bem_near_list(mesh, gg, opts=o)
        nat.nat_bem_assemble(mesh, gg, nl, 2.0, prec="fp32", opts=o)


def test_galerkin_option_errors():
    nat = _nat()
    m = I.icosphere(1)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    o = nat.quad_opts(galerkin=True, ss_order=9)
    nl = nat.nat_bem_near_list(mesh, gg, opts=o)
    with pytest.raises(nat.NatError, match="ss_order"):
        nat.nat_bem_assemble(mesh, gg, nl, 2.0, prec="fp32", opts=o)
