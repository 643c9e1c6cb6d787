"""libnat's kernel timer (nat_kernel_timer_*; bench.py's per-kernel rooflines): one event
pair per main-kernel launch on the launching stream, GMRES launches enqueued after
convergence (which return at once) excluded, algorithmic pairs counted per launch."""
import pytest
import torch

import nat_inputs as I
from gpu_util import requires_cuda

pytestmark = [pytest.mark.gpu, requires_cuda]


def test_kernel_timer_counts_mc_operator_and_far_launches():
    from paper_2506_06190_b200 import nat
    m = I.icosphere(3)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    g = torch.from_numpy(I.neumann_constant(m)[None]).cuda()
    M = 2000
    nat.nat_kernel_timer_enable(True)
    _, _, _, infos = nat.nat_mc_surface_pressure(mesh, geo, [2.0], g, M, seed=3)
    near = nat.nat_bem_near_list(mesh, geo)
    nat.nat_bem_assemble(mesh, geo, near, 2.0, g, prec="fp32")
    sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_MC_OP)
    assert n == infos[0]["iters"] and sec > 0
    assert pairs == n * M * (M - 1)
    assert nat.nat_kernel_timer_read(nat.KTIMER_MC_OP, 1) == (sec, pairs, n)   # one wavenumber per launch
    assert nat.nat_kernel_timer_read(nat.KTIMER_MC_OP, 2)[2] == 0
    sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_MC_RHS)
    assert n == 1 and pairs == M * (M - 1)
    sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_FAR)
    assert n == 1 and pairs == m.n_tri * m.n_tri * 3 and sec > 0
    nat.nat_kernel_timer_enable(False)
    nat.nat_mc_surface_pressure(mesh, geo, [2.0], g, M, seed=3)
    assert nat.nat_kernel_timer_read(nat.KTIMER_MC_OP)[2] == 0   # off: nothing recorded
