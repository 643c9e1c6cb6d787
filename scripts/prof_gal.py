"""Galerkin assembly launches at the C2 shape (icosphere L5, ka = 8, fp32) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

m = I.icosphere(5)
mesh = nat.Mesh.from_numpy(m.v, m.t)
geo = nat.nat_mesh_prepare(mesh)
o = nat.quad_opts(galerkin=True)
near = nat.nat_bem_near_list(mesh, geo, opts=o)
g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
A = torch.empty(m.n_tri, m.n_tri, dtype=torch.complex64, device="cuda")
for _ in range(2):
    nat.nat_bem_assemble(mesh, geo, near, 8.0, g, prec="fp32", A=A, opts=o)
torch.cuda.synchronize()
print("ok")
