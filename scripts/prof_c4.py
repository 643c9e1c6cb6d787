"""One C4 geometry (bowl over slab, M = 2048, 64 wavenumbers): MC solve + 64-mode
radiation to the 64^3 grid, for launch lists / ncu.  argv[1] = geometry index."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

nat.sweep_tuning()   # the bench's configuration

gi = int(sys.argv[1]) if len(sys.argv) > 1 else 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m, g8, D = I.c4_geometry(gi)
ks = list(I.c4_wavenumbers(D))
mesh = nat.Mesh.from_numpy(m.v, m.t)
g = torch.from_numpy(np.tile(g8, (8, 1))).cuda()
M = 2048
plan = nat.McPlan(M, 64, "fp32", 200, "cuda")
P = 64 ** 3
rplan = nat.RadiatePlan(M, 64, P, "fp32", "cuda")
out = torch.empty(64, P, dtype=torch.complex128, device="cuda")
for rep in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    geo = nat.nat_mesh_prepare(mesh)
    smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, ks, g, M, seed=I.SEED, stream_id=gi, prec="fp32",
                                                      plan=plan)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    src = nat.nat_mc_sources(smp, geo.total_area, p, nat.nat_mc_gather_neumann(g, stri), center=geo.center)
    lis = nat.nat_listener_grid(geo.center, geo.bound_radius, 64, 64, 64)
    nat.nat_radiate_field(src, ks, lis, "fp32", out=out, plan=rplan)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    it = [i["iters"] for i in infos]
    print(f"rep {rep}: mc {1e3 * (t1 - t0):.1f} ms (iters min {min(it)} mean {np.mean(it):.1f} max {max(it)}, "
          f"op {1e3 * infos[0]['t_matvec_s']:.1f} ms), radiate {1e3 * (t2 - t1):.1f} ms", flush=True)
