"""NEXT-1, Burton-Miller dense BEM (Eq. BM as printed, beta = i/k; reading R-bm): the CUDA
assembly (far, near and self kernels with the hypersingular and adjoint double-layer
terms) against oracle.bem.assemble(bm=True), and the solve at the fictitious wavenumber
ka = pi where the CBIE fails."""
import math

import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import rel_l2, requires_cuda, to_np
from oracle import analytic, bem, geometry, gmres, nearlist

pytestmark = [pytest.mark.gpu, requires_cuda]

TOL = {"fp32": 1e-4, "fp64": 1e-10}


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name,k", [("ico2", 1.0), ("bowl", math.pi)])
def test_bm_assembly_parity(prec, name, k):
    nat = _nat()
    m = I.icosphere(2) if name == "ico2" else I.bowl(32, 8, 2)
    geo = geometry.mesh_prepare(m.v, m.t)
    near = nearlist.near_list(m.t, geo["centroid"], geo["diam"])
    g = np.stack([I.neumann_rigid_z(m), I.neumann_harmonics(m, 3)[2]])
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, k, g, near=near, bm=True)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    A, b = nat.nat_bem_assemble(mesh, gg, nl, k, torch.from_numpy(g).cuda(), prec=prec,
                                opts=nat.quad_opts(burton_miller=True))
    A = to_np(A)[:, : m.n_tri].astype(np.complex128)
    assert rel_l2(A, A_ref) <= TOL[prec]
    for q in range(2):
        assert rel_l2(to_np(b[q]), b_ref[q]) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_bm_fictitious_frequency_solve(prec):
    """Pulsating sphere at ka = pi (j_0(pi) = 0): the GPU Burton-Miller solution matches the
    oracle's and the analytic p(a) = g a / (ika - 1) within 3 %."""
    nat = _nat()
    m = I.icosphere(3)
    geo = geometry.mesh_prepare(m.v, m.t)
    k = math.pi
    g = np.ones((1, m.n_tri))
    A_ref, b_ref = bem.assemble(m.v, m.t, geo, k, g, bm=True)
    x_ref = np.linalg.solve(A_ref, b_ref[0])
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    A, b = nat.nat_bem_assemble(mesh, gg, nl, k, torch.from_numpy(g).cuda(), prec=prec,
                                opts=nat.quad_opts(burton_miller=True))
    x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6 if prec == "fp32" else 1e-12)
    assert info["converged"] == 1
    x = to_np(x)
    assert rel_l2(x, x_ref) <= (1e-4 if prec == "fp32" else 1e-10)
    exact = analytic.pulsating_sphere(1.0, k)
    assert abs(x.mean() - exact) / abs(exact) < 0.03


def test_bm_requires_positive_k():
    nat = _nat()
    from paper_2506_06190_b200.nat import NatError
    m = I.icosphere(1)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    gg = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, gg)
    with pytest.raises(NatError):
        nat.nat_bem_assemble(mesh, gg, nl, 0.0, None, prec="fp64", opts=nat.quad_opts(burton_miller=True))
