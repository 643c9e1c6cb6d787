"""MC operator launches at the C2 bench shape (M = 10,000; 1 and 3 systems) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

m = I.icosphere(5)
mesh = nat.Mesh.from_numpy(m.v, m.t)
geo = nat.nat_mesh_prepare(mesh)
smp, stri = nat.nat_mc_sample(mesh, geo, 10000, 20250606)
area = geo.total_area
p1 = torch.ones(1, 10000, dtype=torch.complex128, device="cuda")
p3 = torch.ones(3, 10000, dtype=torch.complex128, device="cuda")
for rep in range(2):
    nat.nat_mc_apply(smp, [8.0], p1, area, 0.0, "fp32")
    nat.nat_mc_apply(smp, [0.5, 2.0, 8.0], p3, area, 0.0, "fp32")
torch.cuda.synchronize()
print("ok")
