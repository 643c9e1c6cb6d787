"""Quick timing of nat_radiate_field at the C2 / C3 / C4 launch shapes (dev tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat


def run(m, n_modes, n_lis_dims, ks, prec="fp32", reps=10):
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    p = torch.from_numpy(I.random_complex((n_modes, m.n_tri), 1)).cuda()
    g = torch.from_numpy(I.random_complex((n_modes, m.n_tri), 2)).cuda()
    src = nat.nat_bem_sources(mesh, geo, p, g)
    lis = nat.nat_listener_grid(geo.center, geo.bound_radius, *n_lis_dims)
    plan = nat.RadiatePlan(src.xyz.shape[1], n_modes, lis.shape[1], prec)
    out = nat.nat_radiate_field(src, ks, lis, prec, plan=plan)
    for _ in range(3):
        nat.nat_radiate_field(src, ks, lis, prec, out=out, plan=plan)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nat.nat_radiate_field(src, ks, lis, prec, out=out, plan=plan)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = src.xyz.shape[1] * lis.shape[1] * n_modes
    print(f"{prec} S={src.xyz.shape[1]} P={lis.shape[1]} modes={n_modes}: {ms:.3f} ms "
          f"-> {pairs / ms / 1e9:.1f} Tpair/s ({pairs/ms/1e9/1.551:.1%} of R_pipe@1965)")


if __name__ == "__main__":
    run(I.icosphere(5), 1, (32, 32, 32), [8.0])
    run(I.icosphere(5), 3, (32, 32, 32), [0.5, 2.0, 8.0])
    run(I.bowl(), 32, (32, 32, 32), list(I.c3_wavenumbers()), reps=3)
    m, g, D = I.c4_geometry(0)
    run(m, 64, (64, 64, 64), list(I.c4_wavenumbers(D)), reps=2)
    run(I.icosphere(5), 1, (32, 32, 32), [8.0], prec="fp64", reps=2)
