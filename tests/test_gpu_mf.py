"""NEXT-3: the matrix-free dense BEM operator (nat_bem_mf_*) against the
oracle's stored operator (oracle/bem.py assemble, the same A of P:174-191 with the rules
of reading R-colloc), and the C5 mesh solved on ONE GPU (its stored matrix would be
638 GB) against the oracle's rows and the analytic oscillating sphere (≤ 2 %)."""
import functools

import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import rel_l2, requires_cuda, soa_to_aos, to_np
from oracle import analytic, bem, geometry, nearlist

pytestmark = [pytest.mark.gpu, requires_cuda]

TOL = {"fp32": 1e-4, "fp64": 1e-10}


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


@functools.lru_cache(maxsize=None)
def _oracle_ico3(k):
    m = I.icosphere(3)
    geo = geometry.mesh_prepare(m.v, m.t)
    near = nearlist.near_list(m.t, geo["centroid"], geo["diam"])
    g = I.neumann_rigid_z(m)
    A, b = bem.assemble(m.v, m.t, geo, k, g[None], near=near)
    return m, g, A, b


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("k", [1.0, 4.0])
def test_mf_matvec_and_rhs_full(prec, k):
    """Whole C1-size operator: (A x) and rhs = -V g element by element."""
    nat = _nat()
    m, g, A_r, b_r = _oracle_ico3(k)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    op, rhs = nat.nat_bem_mf_prepare(mesh, gg, nl, k, torch.from_numpy(g[None]).cuda(), prec=prec)
    assert rel_l2(to_np(rhs[0]), b_r[0]) <= TOL[prec]
    for seed in (3, 4):
        x = I.random_complex(m.n_tri, seed)
        y = to_np(nat.nat_bem_mf_matvec(op, torch.from_numpy(x).cuda()))
        assert rel_l2(y, A_r @ x) <= TOL[prec]
    # same operator as the stored path (the matrix-free far sums run in another order)
    A, _ = nat.nat_bem_assemble(mesh, gg, nl, k, prec=prec)
    x = torch.from_numpy(I.random_complex(m.n_tri, 5)).cuda()
    ys = to_np(nat.nat_bem_matvec(A, x, n=m.n_tri))
    assert rel_l2(to_np(nat.nat_bem_mf_matvec(op, x)), ys) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_mf_row_blocks_ragged(prec):
    """Row blocks of a 3-way split (ragged last block, as rank r of 3 owns them) give the
    oracle's rows; the zero vector maps to zero."""
    nat = _nat()
    k = 2.0
    m, g, A_r, b_r = _oracle_ico3(k)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    x = I.random_complex(m.n_tri, 9)
    xt = torch.from_numpy(x).cuda()
    ys = []
    for r in range(3):
        r0, r1 = nat.row_range(m.n_tri, r, 3)
        nl = nat.nat_bem_near_list(mesh, gg, r0, r1)
        op, rhs = nat.nat_bem_mf_prepare(mesh, gg, nl, k, torch.from_numpy(g[None]).cuda(), prec=prec)
        y = to_np(nat.nat_bem_mf_matvec(op, xt))
        assert rel_l2(y, A_r[r0:r1] @ x) <= TOL[prec]
        assert rel_l2(to_np(rhs[0]), b_r[0, r0:r1]) <= TOL[prec]
        assert np.all(to_np(nat.nat_bem_mf_matvec(op, torch.zeros_like(xt))) == 0)
        ys.append(y)
    # the far sums are reduced in fixed column blocks: a row's value does not depend on the split
    nl = nat.nat_bem_near_list(mesh, gg)
    op, _ = nat.nat_bem_mf_prepare(mesh, gg, nl, k, prec=prec)
    assert np.array_equal(np.concatenate(ys), to_np(nat.nat_bem_mf_matvec(op, xt)))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_mf_solve_matches_oracle_solution(prec):
    nat = _nat()
    k = 1.0
    m, g, A_r, b_r = _oracle_ico3(k)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    op, rhs = nat.nat_bem_mf_prepare(mesh, gg, nl, k, torch.from_numpy(g[None]).cuda(), prec=prec)
    tol = 1e-6 if prec == "fp32" else 1e-12
    x, info = nat.nat_bem_mf_solve(op, rhs[0], tol=tol)
    assert info["converged"] == 1 and info["rel_residual"] <= tol * 1.01
    x_r = np.linalg.solve(A_r, b_r[0])
    assert rel_l2(to_np(x), x_r) <= TOL[prec]
    # same iterate as the stored-matrix solve
    A, b = nat.nat_bem_assemble(mesh, gg, nl, k, torch.from_numpy(g[None]).cuda(), prec=prec)
    xs, info_s = nat.nat_bem_solve(A, b[0], m.n_tri, tol=tol)
    assert abs(info_s["iters"] - info["iters"]) <= 1
    assert rel_l2(to_np(x), to_np(xs)) <= TOL[prec]


def test_mf_rejects_burton_miller_and_host_pointers():
    nat = _nat()
    m = I.icosphere(2)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    with pytest.raises(nat.NatError, match="conventional BIE"):
        nat.nat_bem_mf_prepare(mesh, gg, nl, 2.0, opts=nat.quad_opts(burton_miller=True))
    op, _ = nat.nat_bem_mf_prepare(mesh, gg, nl, 2.0)
    with pytest.raises(nat.NatError):
        nat.nat_bem_mf_matvec(op, torch.zeros(m.n_tri, dtype=torch.complex128))


def test_c2_mf_fp32_sampled_rows():
    """C2 launch shape (icosphere L5, 20,480 tri, ka = 8, fp32): sampled rows of the
    matrix-free product and rhs against the oracle's rows."""
    nat = _nat()
    ka = 8.0
    m = I.icosphere(5)
    g = I.neumann_rigid_z(m)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    op, rhs = nat.nat_bem_mf_prepare(mesh, gg, nl, ka, torch.from_numpy(g[None]).cuda(), prec="fp32")
    x = I.random_complex(m.n_tri, 11)
    y = to_np(nat.nat_bem_mf_matvec(op, torch.from_numpy(x).cuda()))
    geo = geometry.mesh_prepare(m.v, m.t)
    rows = np.random.default_rng(2).choice(m.n_tri, 6, replace=False)
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, ka, g[None], rows=rows)
    assert rel_l2(y[rows], A_ref @ x) <= 1e-4
    assert rel_l2(to_np(rhs[0])[rows], b_ref[0]) <= 1e-4


def test_c5_matrix_free_fp64_solve_one_gpu():
    """C5 (equiangular cubed sphere, 199,692 tri, dipole, ka = 8, fp64, tol 1e-12) solved
    on one GPU without storing A: sampled rows of A x and b against the oracle's rows
    (1e-10), and the radiated field against the analytic oscillating sphere (≤ 2 %)."""
    nat = _nat()
    ka = 8.0
    m = I.cubed_sphere(129)
    g = I.neumann_rigid_z(m)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    gt = torch.from_numpy(g[None]).cuda()
    op, rhs = nat.nat_bem_mf_prepare(mesh, gg, nl, ka, gt, prec="fp64")
    x, info = nat.nat_bem_mf_solve(op, rhs[0], tol=1e-12)
    assert info["converged"] == 1 and info["rel_residual"] <= 1.01e-12
    geo = geometry.mesh_prepare(m.v, m.t)
    rows = np.array([0, 54_321, 123_456, 199_691])
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, ka, g[None], rows=rows)
    assert rel_l2(to_np(rhs[0])[rows], b_ref[0]) <= 1e-10
    xs = to_np(x)
    y = to_np(nat.nat_bem_mf_matvec(op, x))
    assert rel_l2(y[rows], A_ref @ xs) <= 1e-10
    assert np.linalg.norm(A_ref @ xs - b_ref[0]) / np.linalg.norm(b_ref[0]) <= 1e-10
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 8, 8, 4)
    src = nat.nat_bem_sources(mesh, gg, x[None], gt)
    p = to_np(nat.nat_radiate_field(src, [ka], lis, "fp64"))[0]
    pe = analytic.oscillating_sphere(soa_to_aos(lis), ka)
    assert rel_l2(p, pe) <= 0.02
