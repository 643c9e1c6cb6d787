"""Rows a2 (near list), a4+a5 (assembly), a6 (matvec), a7 (GMRES) and the full dense
BEM path (C1 end to end, C2 launch configuration on sampled rows): CUDA vs oracle."""
import functools

import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import rel_l2, requires_cuda, soa_to_aos, to_np
from oracle import analytic, bem, geometry, gmres, listeners, nearlist, radiate

pytestmark = [pytest.mark.gpu, requires_cuda]

TOL = {"fp32": 1e-4, "fp64": 1e-10}


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


@functools.lru_cache(maxsize=None)
def _oracle_case(name):
    m = {"ico2": lambda: I.icosphere(2), "ico3": lambda: I.icosphere(3),
         "bowl": lambda: I.bowl(32, 8, 2)}[name]()
    geo = geometry.mesh_prepare(m.v, m.t)
    near = nearlist.near_list(m.t, geo["centroid"], geo["diam"])
    return m, geo, near


def _gpu_case(m):
    nat = _nat()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    return mesh, nat.nat_mesh_prepare(mesh)


@pytest.mark.parametrize("name", ["ico3", "bowl"])
def test_near_list_bitwise(name):
    nat = _nat()
    m, geo, (rp, col, cls) = _oracle_case(name)
    mesh, g = _gpu_case(m)
    nl = nat.nat_bem_near_list(mesh, g)
    assert np.array_equal(to_np(nl.row_ptr), rp)
    assert np.array_equal(to_np(nl.col), col)
    assert np.array_equal(to_np(nl.cls), cls)


def test_near_list_row_range_and_c4_scene():
    nat = _nat()
    m = I.c4_geometry(3)[0]
    geo = geometry.mesh_prepare(m.v, m.t)
    rows = np.arange(7000, 7400)              # bowl/slab boundary region of the scene
    rp, col, cls = nearlist.near_list(m.t, geo["centroid"], geo["diam"], rows=rows)
    mesh, g = _gpu_case(m)
    nl = nat.nat_bem_near_list(mesh, g, 7000, 7400)
    assert np.array_equal(to_np(nl.row_ptr), rp)
    assert np.array_equal(to_np(nl.col), col)
    assert np.array_equal(to_np(nl.cls), cls)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name,k", [("ico2", 2.0), ("bowl", 5.0), ("ico3", 1.0)])
def test_assembly_parity(prec, name, k):
    nat = _nat()
    m, geo, near = _oracle_case(name)
    g = np.stack([I.neumann_rigid_z(m), I.random_complex(m.n_tri, 3)])
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, k, g, near=near)
    mesh, gg = _gpu_case(m)
    nl = nat.nat_bem_near_list(mesh, gg)
    A, b = nat.nat_bem_assemble(mesh, gg, nl, k, torch.from_numpy(g).cuda(), prec=prec)
    A = to_np(A)[:, : m.n_tri]
    assert rel_l2(A, A_ref) <= TOL[prec]
    for q in range(2):
        assert rel_l2(to_np(b)[q], b_ref[q]) <= TOL[prec]
    # every row individually (catches a wrong near/self entry hidden by the global norm)
    rows = np.linalg.norm(A - A_ref, axis=1) / np.linalg.norm(A_ref, axis=1)
    assert rows.max() <= 10 * TOL[prec]


def test_assembly_row_ranges_match_full_and_odd_lda():
    nat = _nat()
    m, geo, near = _oracle_case("ico2")
    mesh, gg = _gpu_case(m)
    g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
    full = nat.nat_bem_near_list(mesh, gg)
    A_full, b_full = nat.nat_bem_assemble(mesh, gg, full, 3.0, g, prec="fp64")
    parts_A, parts_b = [], []
    for r0, r1 in ((0, 101), (101, 250), (250, m.n_tri)):
        nl = nat.nat_bem_near_list(mesh, gg, r0, r1)
        A, b = nat.nat_bem_assemble(mesh, gg, nl, 3.0, g, prec="fp64", lda=m.n_tri + 5)
        parts_A.append(A[:, : m.n_tri])
        parts_b.append(b)
    assert torch.equal(torch.cat(parts_A), A_full[:, : m.n_tri])
    assert torch.equal(torch.cat(parts_b, dim=1), b_full)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_matvec_parity(prec):
    nat = _nat()
    rng = np.random.default_rng(0)
    for rows, n in ((1, 1), (13, 1001), (517, 4099)):
        A = I.random_complex((rows, n + 1), rows)
        x = I.random_complex(n, n)
        dt = torch.complex64 if prec == "fp32" else torch.complex128
        At = torch.from_numpy(A).to(dt).cuda()
        y = to_np(nat.nat_bem_matvec(At, torch.from_numpy(x).cuda(), n=n))
        Aq = to_np(At).astype(np.complex128)[:, :n]      # the stored (rounded) matrix
        # fp64: fp64 products; fp32 (c64 matrix): fp32 products flushed to fp64 every 16
        assert rel_l2(y, Aq @ x) <= (1e-13 if prec == "fp64" else 1e-6)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_gmres_parity_and_contract(prec):
    nat = _nat()
    n = 300
    rng = np.random.default_rng(4)
    A = np.eye(n) + 0.3 * (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    dt = torch.complex64 if prec == "fp32" else torch.complex128
    At = torch.from_numpy(A).to(dt).cuda()
    Aq = to_np(At).astype(np.complex128)
    tol = 1e-6 if prec == "fp32" else 1e-12
    x, info = nat.nat_bem_solve(At, torch.from_numpy(b).cuda(), n, tol=tol)
    xo, io = gmres.gmres(lambda z: Aq @ z, b, tol=1e-13, max_iter=300)
    assert info["converged"] == 1 and info["rel_residual"] <= tol
    assert rel_l2(to_np(x), xo) <= (1e-5 if prec == "fp32" else 1e-11)
    # the reported residual (b - sum_k y_k A v_k, from the saved operator products) is the
    # true ||b - A x|| / ||b|| up to the matvec rounding (fp32 products: ~1e-7)
    direct = np.linalg.norm(b - Aq @ to_np(x)) / np.linalg.norm(b)
    assert abs(info["rel_residual"] - direct) <= (1e-6 if prec == "fp32" else 1e-13)
    # zero right-hand side -> 0 iterations, x = 0
    x0, i0 = nat.nat_bem_solve(At, torch.zeros(n, dtype=torch.complex128, device="cuda"), n)
    assert i0["iters"] == 0 and torch.count_nonzero(x0) == 0
    # non-convergence is a warning with the best iterate
    x3, i3 = nat.nat_bem_solve(At, torch.from_numpy(b).cuda(), n, tol=1e-14, max_iter=3)
    assert i3["converged"] == 0 and i3["iters"] == 3 and i3["rel_residual"] < 1.0
    xo3, io3 = gmres.gmres(lambda z: Aq @ z, b, tol=1e-14, max_iter=3)
    assert rel_l2(to_np(x3), xo3) <= 1e-5


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_c1_end_to_end(prec):
    """Config C1: icosphere L3, g = 1, k = 1, 4^3 listeners: parity with the oracle and
    <= 2% against the analytic pulsating sphere."""
    nat = _nat()
    m, geo, near = _oracle_case("ico3")
    k = 1.0
    g = I.neumann_constant(m)
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, k, g[None], near=near)
    x_ref, _ = gmres.gmres(lambda z: A_ref @ z, b_ref[0], tol=1e-12)
    L = listeners.shell_grid(np.zeros(3), 1.0, 4, 4, 4)
    p_ref = radiate.radiate(radiate.bem_sources(m.v, m.t, geo, x_ref[None], g[None]), [k], L)[0]

    mesh, gg = _gpu_case(m)
    nl = nat.nat_bem_near_list(mesh, gg)
    gt = torch.from_numpy(g[None]).cuda()
    A, b = nat.nat_bem_assemble(mesh, gg, nl, k, gt, prec=prec)
    x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6 if prec == "fp32" else 1e-12)
    src = nat.nat_bem_sources(mesh, gg, x[None], gt)
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 4, 4, 4)
    p = to_np(nat.nat_radiate_field(src, [k], lis, prec=prec))[0]
    assert rel_l2(to_np(x), x_ref) <= TOL[prec]
    assert rel_l2(p, p_ref) <= TOL[prec]
    pe = analytic.pulsating_sphere(np.linalg.norm(soa_to_aos(lis), axis=1), k)
    assert rel_l2(p, pe) <= 0.02


@pytest.mark.parametrize("ka", [0.5, 2.0, 8.0])
def test_c2_launch_configuration(ka):
    """Config C2 (icosphere L5, 20,480 tri, dipole) in the launch configuration bench.py
    times: sampled rows of A and b against the oracle, the GPU solution's residual in the
    oracle's own rows, and the radiated field against the analytic dipole (<= 2%)."""
    nat = _nat()
    m = I.icosphere(5)
    g = I.neumann_rigid_z(m)
    mesh, gg = _gpu_case(m)
    nl = nat.nat_bem_near_list(mesh, gg)
    gt = torch.from_numpy(g[None]).cuda()
    A, b = nat.nat_bem_assemble(mesh, gg, nl, ka, gt, prec="fp32")
    x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6)
    assert info["converged"] == 1
    geo = geometry.mesh_prepare(m.v, m.t)
    rows = np.random.default_rng(int(ka * 10)).choice(m.n_tri, 6, replace=False)
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, ka, g[None], rows=rows)
    A_rows = to_np(A[torch.from_numpy(rows).cuda()])[:, : m.n_tri].astype(np.complex128)
    assert rel_l2(A_rows, A_ref) <= 1e-4
    assert rel_l2(to_np(b[0])[rows], b_ref[0]) <= 1e-4
    xs = to_np(x)
    res = A_ref @ xs - b_ref[0]
    assert np.linalg.norm(res) / np.linalg.norm(b_ref[0]) <= 1e-4
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 32, 32, 32)
    src = nat.nat_bem_sources(mesh, gg, x[None], gt)
    p = to_np(nat.nat_radiate_field(src, [ka], lis))[0]
    pe = analytic.oscillating_sphere(soa_to_aos(lis), ka)
    assert rel_l2(p, pe) <= 0.02


def test_borrowed_single_rank_communicator_matches_no_communicator():
    """nat_comm_create with a NULL ncclComm_t (world 1): the row-sharded solve with a
    borrowed communicator equals the solve without one, bit for bit."""
    nat = _nat()
    m = I.icosphere(3)
    g = I.neumann_rigid_z(m)
    mesh, gg = _gpu_case(m)
    nl = nat.nat_bem_near_list(mesh, gg)
    A, b = nat.nat_bem_assemble(mesh, gg, nl, 2.0, torch.from_numpy(g[None]).cuda(), prec="fp32")
    x0, i0 = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6)
    comm = nat.Comm.borrow(None)
    x1, i1 = nat.nat_bem_solve(A, b[0], m.n_tri, comm=comm, tol=1e-6)
    comm.close()
    assert i0["iters"] == i1["iters"] and torch.equal(x0, x1)
    with pytest.raises(nat.NatError):
        nat.Comm.borrow(None, 0, 2)     # a NULL ncclComm_t cannot have two ranks


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("far_pts", [1, 6, 7])
def test_assembly_other_far_rules(prec, far_pts):
    """nat_quad_opts.far_pts 1 / 6 / 7 (R-colloc): the 1- and 7-point rules contain the
    centroid, i.e. the row's own collocation point, so the far rule is singular on the self
    pair; the far kernels zero it and the self kernel adds the exact polar value.  Parity
    with the oracle using the same rule, and finite everywhere (matrix-free operator too)."""
    nat = _nat()
    m, geo, near = _oracle_case("ico2")
    g = I.neumann_rigid_z(m)[None]
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, 2.0, g, near=near, opts=dict(far_pts=far_pts))
    mesh, gg = _gpu_case(m)
    o = nat.quad_opts(far_pts=far_pts)
    nl = nat.nat_bem_near_list(mesh, gg, opts=o)
    A, b = nat.nat_bem_assemble(mesh, gg, nl, 2.0, torch.from_numpy(g).cuda(), prec=prec, opts=o)
    A = to_np(A)[:, : m.n_tri]
    assert np.all(np.isfinite(A)) and np.all(np.isfinite(to_np(b)))
    assert rel_l2(A, A_ref) <= TOL[prec]
    assert rel_l2(to_np(b)[0], b_ref[0]) <= TOL[prec]
    op, rhs = nat.nat_bem_mf_prepare(mesh, gg, nl, 2.0, torch.from_numpy(g).cuda(), prec=prec, opts=o)
    x = I.random_complex(m.n_tri, 4)
    y = to_np(nat.nat_bem_mf_matvec(op, torch.from_numpy(x).cuda()))
    assert np.all(np.isfinite(y)) and rel_l2(y, A_ref @ x) <= TOL[prec]
    assert rel_l2(to_np(rhs)[0], b_ref[0]) <= TOL[prec]


@pytest.mark.parametrize("prec,n_rhs,far_pts", [("fp32", 1, 3), ("fp32", 0, 7), ("fp32", 2, 3), ("fp64", 1, 3)])
def test_assemble_multi_equals_single_calls(prec, n_rhs, far_pts):
    """nat_bem_assemble_multi (one far pass for several wavenumbers on the fp32 collocation
    path, a loop elsewhere) writes exactly what separate nat_bem_assemble calls write."""
    nat = _nat()
    m, geo, near = _oracle_case("bowl")
    mesh, gg = _gpu_case(m)
    o = nat.quad_opts(far_pts=far_pts)
    nl = nat.nat_bem_near_list(mesh, gg, 37, m.n_tri - 11, opts=o)     # a ragged row block
    ks = [0.5, 2.0, 8.0]
    g = torch.from_numpy(np.stack([I.neumann_rigid_z(m), I.random_complex(m.n_tri, 5)])[:n_rhs]).cuda() if n_rhs else None
    As, rhs = nat.nat_bem_assemble_multi(mesh, gg, nl, ks, g, prec=prec, opts=o)
    for q, k in enumerate(ks):
        A1, b1 = nat.nat_bem_assemble(mesh, gg, nl, k, g, prec=prec, opts=o)
        assert torch.equal(As[q], A1), (q, k)
        if n_rhs:
            assert torch.equal(rhs[q], b1), (q, k)
