"""Launch-shape sweep of the fp32 pair kernels at the C4 shapes (kernel timer, no ncu):
MC operator (kind 1) and right-hand side (kind 2) at M = 2048 with 64 / 16 / 4 systems,
radiation (kind 0) of 64 modes from 2048 sources to 64^3 listeners.  Prints the kernel's
pair-evals x wavenumbers per second for each R, NT, chunk, MB (NAT_RAD_PLAN override)."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

m, g8, D = I.c4_geometry(0)
ks = list(I.c4_wavenumbers(D))
mesh = nat.Mesh.from_numpy(m.v, m.t)
geo = nat.nat_mesh_prepare(mesh)
M = 2048
smp, stri = nat.nat_mc_sample(mesh, geo, M, 20250606, 0)
lis = nat.nat_listener_grid(geo.center, geo.bound_radius, 64, 64, 64)
which = sys.argv[1:] or ["op64", "op16", "op4", "rhs64", "rad64"]


def run(case):
    if case.startswith("op"):
        ns = int(case[2:])
        p = torch.ones(ns, M, dtype=torch.complex128, device="cuda")
        nat.nat_mc_apply(smp, ks[:ns], p, geo.total_area)
        return nat.KTIMER_MC_OP
    if case.startswith("rhs"):
        ns = int(case[3:])
        g = torch.ones(ns, M, dtype=torch.complex128, device="cuda")
        nat.nat_mc_rhs(smp, ks[:ns], g, geo.total_area)
        return nat.KTIMER_MC_RHS
    p = torch.ones(64, M, dtype=torch.complex128, device="cuda")
    src = nat.nat_mc_sources(smp, geo.total_area, p, p, center=geo.center)
    nat.nat_radiate_field(src, ks, lis, "fp32")
    return nat.KTIMER_RADIATE


for case in which:
    res = []
    os.environ.pop("NAT_RAD_PLAN", None)
    run(case)
    nat.nat_kernel_timer_enable(True)
    cat = run(case)
    sec, pairs, n = nat.nat_kernel_timer_read(cat)
    nat.nat_kernel_timer_enable(False)
    print(f"{case} default: {pairs / sec / 1e9:.0f} Gpair/s", flush=True)
    for R, NT, c, MB in itertools.product((2, 4), (128, 256), (1, 2, 4, 8), (4, 8)):
        os.environ["NAT_RAD_PLAN"] = f"{R},{NT},{c},{MB}"
        try:
            run(case)
            nat.nat_kernel_timer_enable(True)
            for _ in range(3):
                cat = run(case)
            sec, pairs, n = nat.nat_kernel_timer_read(cat)
            nat.nat_kernel_timer_enable(False)
            res.append((pairs / sec / 1e9, R, NT, c, MB))
        except Exception as ex:
            nat.nat_kernel_timer_enable(False)
            print(case, R, NT, c, MB, "error", ex)
    res.sort(reverse=True)
    for r in res[:6]:
        print(f"{case} R {r[1]} NT {r[2]} c {r[3]} MB {r[4]}: {r[0]:.0f} Gpair/s", flush=True)
os.environ.pop("NAT_RAD_PLAN", None)
