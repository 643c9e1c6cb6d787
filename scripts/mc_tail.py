"""One C4 geometry's MC solve (serial): MC-operator launches bucketed by the number of
active wavenumbers n (kernel timer), each bucket's time and fraction of R(n)."""
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
R = lambda n: 16 * 148 * 1.965e9 / (2 + 1 / n)
for rep in range(2):
    torch.cuda.synchronize()
    nat.nat_kernel_timer_enable(True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, ks, g, 2048, seed=I.SEED, stream_id=gi, prec="fp32",
                                                      plan=plan)
    ev[1].record()
    torch.cuda.synchronize()
    call = ev[0].elapsed_time(ev[1]) * 1e-3
    rows, tot_t, tot_ideal = [], 0.0, 0.0
    for n in range(1, 65):
        s, pr, c = nat.nat_kernel_timer_read(nat.KTIMER_MC_OP, n)
        if c:
            rows.append((n, c, s, pr, pr / R(n)))
            tot_t += s
            tot_ideal += pr / R(n)
    sr, prr, _ = nat.nat_kernel_timer_read(nat.KTIMER_MC_RHS)
    nat.nat_kernel_timer_enable(False)
it = sorted(i["iters"] for i in infos)
print("iters", it)
print(" n launches   ms     Gpairs  frac")
for n, c, s, pr, ideal in rows:
    print(f"{n:2d} {c:5d} {1e3 * s:8.3f} {pr / 1e9:8.2f} {ideal / s:.3f}")
rhs_ideal = prr / R(64)
print(f"op total {1e3 * tot_t:.2f} ms, ideal {1e3 * tot_ideal:.2f} ms, frac {tot_ideal / tot_t:.3f}")
print(f"rhs {1e3 * sr:.3f} ms frac {rhs_ideal / sr:.3f}")
print(f"call {1e3 * call:.2f} ms, call frac {(tot_ideal + rhs_ideal) / call:.3f}")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for rep in range(2):
    ev[0].record()
    nat.nat_mc_surface_pressure(mesh, geo, ks, g, 2048, seed=I.SEED, stream_id=gi, prec="fp32", plan=plan)
    ev[1].record()
    torch.cuda.synchronize()
print(f"call without the kernel timer {ev[0].elapsed_time(ev[1]):.2f} ms, call frac {(tot_ideal + rhs_ideal) / (ev[0].elapsed_time(ev[1]) * 1e-3):.3f}")
