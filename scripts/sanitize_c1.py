"""C1-sized run of the main entry points for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

m = I.icosphere(3)
mesh = nat.Mesh.from_numpy(m.v, m.t)
geo = nat.nat_mesh_prepare(mesh)
near = nat.nat_bem_near_list(mesh, geo)
g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
A, b = nat.nat_bem_assemble(mesh, geo, near, 2.0, g, prec="fp32")
x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6)
smp, tri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, [0.5, 2.0], g.repeat(2, 1), 500, seed=1)
src = nat.nat_mc_sources(smp, geo.total_area, p, nat.nat_mc_gather_neumann(g.repeat(2, 1), tri), center=geo.center)
lis = nat.nat_listener_grid(geo.center, geo.bound_radius, 8, 8, 8)
f = nat.nat_radiate_field(src, [0.5, 2.0], lis)
torch.cuda.synchronize()
print("ok", float(x.abs().sum()), float(f.abs().sum()))
