"""Matrix-free far-kernel launches for ncu: fp32 at C2 (icosphere L5, all rows) and fp64 on
a 2048-row block of the C5 cubed sphere (the kernel of the one-GPU C5 solve)."""
import sys

import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

for m, prec, r1 in ((I.icosphere(5), "fp32", None), (I.cubed_sphere(129), "fp64", 2048)):
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    nl = nat.nat_bem_near_list(mesh, geo, 0, r1 or m.n_tri)
    op, _ = nat.nat_bem_mf_prepare(mesh, geo, nl, 8.0, prec=prec)
    x = torch.from_numpy(I.random_complex(m.n_tri, 1)).cuda()
    for _ in range(2):
        nat.nat_bem_mf_matvec(op, x)
torch.cuda.synchronize()
print("ok")
