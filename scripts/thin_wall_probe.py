"""Thin-wall point-source probe (C3 acceptance): dense BEM fp64 errors at
3,200 and 12,544 triangles and MC statistics, to set the GPU test tolerances."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import nat_inputs as I
from oracle import analytic, listeners
from paper_2506_06190_b200 import nat

xs, k = np.array([0.0, 0.0, -0.95]), 2.0
for na, npsi in ((64, 12), (128, 24)):
    m = I.bowl(na, npsi, 2)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    c = geo.centroid.T.cpu().numpy(); nn = geo.normal.T.cpu().numpy()
    g = torch.from_numpy(analytic.point_source_dn(c, nn, xs, k)[None]).cuda()
    near = nat.nat_bem_near_list(mesh, geo)
    A, b = nat.nat_bem_assemble(mesh, geo, near, k, g, prec="fp64")
    x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-12)
    L = listeners.shell_grid(np.array(geo.center), geo.bound_radius, 8, 8, 4)
    lis = torch.from_numpy(np.ascontiguousarray(L.T)).cuda()
    p = nat.nat_radiate_field(nat.nat_bem_sources(mesh, geo, x[None], g), [k], lis, "fp64")[0].cpu().numpy()
    pe = analytic.point_source(L, xs, k)
    print(m.n_tri, "dense fp64 field err", np.linalg.norm(p - pe) / np.linalg.norm(pe), "iters", info["iters"], flush=True)
    if na == 128:
        for M in (2048, 4096, 8192):
            errs, fields = [], []
            for seed in range(4):
                smp, stri, pm, inf = nat.nat_mc_surface_pressure(mesh, geo, [k], g, M, seed=seed, prec="fp32")
                gs = nat.nat_mc_gather_neumann(g, stri)
                f = nat.nat_radiate_field(nat.nat_mc_sources(smp, geo.total_area, pm, gs, center=geo.center), [k], lis)[0].cpu().numpy()
                fields.append(f)
                errs.append(np.linalg.norm(f - pe) / np.linalg.norm(pe))
            fm = np.mean(fields, axis=0)
            print(M, "MC per-seed errs", np.round(errs, 4), "seed-mean field err", np.linalg.norm(fm - pe) / np.linalg.norm(pe), flush=True)
