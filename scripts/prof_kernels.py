"""Runs each hot kernel of the C2 step once (after a warm-up) so ncu can capture them:
far/near/self assembly, GEMV (via a 2-iteration solve), BEM radiation, MC operator."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat


def main():
    m = I.icosphere(5)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    near = nat.nat_bem_near_list(mesh, geo)
    g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 32, 32, 32)
    for rep in range(2):  # rep 0 = warm-up, rep 1 = the captured launches
        A, b = nat.nat_bem_assemble(mesh, geo, near, 8.0, g, prec="fp32")
        x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6, max_iter=3)
        x3 = torch.stack([x, x, x])
        src = nat.nat_bem_sources(mesh, geo, x3, torch.cat([g, g, g]))
        nat.nat_radiate_field(src, [0.5, 2.0, 8.0], lis, "fp32")   # the bench's 3 fused wavenumbers
        smp, stri = nat.nat_mc_sample(mesh, geo, 10000, 20250606)
        area = geo.total_area
        p = torch.ones(3, 10000, dtype=torch.complex128, device="cuda")
        nat.nat_mc_apply(smp, [0.5, 2.0, 8.0], p, area, 0.0, "fp32")
        nat.nat_mc_apply(smp, [8.0], p[:1], area, 0.0, "fp32")
        nat.nat_mc_rhs(smp, [0.5, 2.0, 8.0], p, area, 0.0, "fp32")
        torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
