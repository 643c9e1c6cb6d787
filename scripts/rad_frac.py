"""C4 radiation (64 wavenumbers, 2048 MC sources -> 64^3 listeners) and MC operator: kernel-timer
fraction of R(n) for one geometry (3 repetitions)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

m, g8, D = I.c4_geometry(0)
ks = list(I.c4_wavenumbers(D))
mesh = nat.Mesh.from_numpy(m.v, m.t)
g = torch.from_numpy(np.tile(g8, (8, 1))).cuda()
geo = nat.nat_mesh_prepare(mesh)
plan = nat.McPlan(2048, 64, "fp32", 200, "cuda")
smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, ks, g, 2048, seed=I.SEED, prec="fp32", plan=plan)
src = nat.nat_mc_sources(smp, geo.total_area, p, nat.nat_mc_gather_neumann(g, stri), center=geo.center)
lis = nat.nat_listener_grid(geo.center, geo.bound_radius, 64, 64, 64)
rplan = nat.RadiatePlan(2048, 64, 64 ** 3, "fp32", "cuda")
out = torch.empty(64, 64 ** 3, dtype=torch.complex128, device="cuda")
R64 = 16 * 148 * 1.965e9 / (2 + 1 / 64)
for rep in range(3):
    nat.nat_kernel_timer_enable(True)
    nat.nat_radiate_field(src, ks, lis, "fp32", out=out, plan=rplan)
    nat.nat_mc_surface_pressure(mesh, geo, ks, g, 2048, seed=I.SEED, prec="fp32", plan=plan)
    torch.cuda.synchronize()
    sec, pairs, _ = nat.nat_kernel_timer_read(nat.KTIMER_RADIATE)
    s64, p64, _ = nat.nat_kernel_timer_read(nat.KTIMER_MC_OP, 32)   # two solve groups of 32
    nat.nat_kernel_timer_enable(False)
    R32 = 16 * 148 * 1.965e9 / (2 + 1 / 32)
    print(f"radiation {1e3 * sec:.2f} ms frac {pairs / sec / R64:.3f}; MC op 32-system launches frac {p64 / s64 / R32:.3f}")
