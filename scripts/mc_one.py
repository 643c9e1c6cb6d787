"""One C4 geometry's MC solve, once (for ncu launch lists of the Krylov iteration)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

gi = int(sys.argv[1]) if len(sys.argv) > 1 else 0
m, g8, D = I.c4_geometry(gi)
ks = list(I.c4_wavenumbers(D))
mesh = nat.Mesh.from_numpy(m.v, m.t)
g = torch.from_numpy(np.tile(g8, (8, 1))).cuda()
plan = nat.McPlan(2048, 64, "fp32", 200, "cuda")
geo = nat.nat_mesh_prepare(mesh)
smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, ks, g, 2048, seed=I.SEED, stream_id=gi, prec="fp32", plan=plan)
torch.cuda.synchronize()
print("iters", sorted(i["iters"] for i in infos))
