"""Sweep of forced launch plans (NAT_RAD_PLAN = "R,NT,c") for the MC operator main kernel
at the C2 bench shape (M = 10,000 samples, 1 and 3 systems), timed with libnat's kernel
timer (CUDA events around the main kernel only)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

m = I.icosphere(5)
mesh = nat.Mesh.from_numpy(m.v, m.t)
geo = nat.nat_mesh_prepare(mesh)
M = 10000
smp, stri = nat.nat_mc_sample(mesh, geo, M, 20250606)
area = geo.total_area
R_PIPE = 148 * 128 * 1965e6 / 24


def run(nsys, plan):
    if plan:
        os.environ["NAT_RAD_PLAN"] = plan
    else:
        os.environ.pop("NAT_RAD_PLAN", None)
    p = torch.ones(nsys, M, dtype=torch.complex128, device="cuda")
    ks = [0.5, 2.0, 8.0][:nsys] if nsys <= 3 else [8.0] * nsys
    for _ in range(2):
        nat.nat_mc_apply(smp, ks, p, area, 0.0, "fp32")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        nat.nat_mc_apply(smp, ks, p, area, 0.0, "fp32")
    e1.record()
    torch.cuda.synchronize()
    t_app = e0.elapsed_time(e1) / 10 * 1e3
    nat.nat_kernel_timer_enable(True)
    for _ in range(10):
        nat.nat_mc_apply(smp, ks, p, area, 0.0, "fp32")
    sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_MC_OP)
    nat.nat_kernel_timer_enable(False)
    return sec / n * 1e6, pairs / sec / R_PIPE, t_app


for nsys in (1, 3):
    t, f, ta = run(nsys, None)
    print(f"nsys={nsys} auto: kernel {t:.1f} us (frac {f:.3f}), application {ta:.1f} us", flush=True)
    res = []
    for R in (2, 4):
        for NT in (128, 256):
            for c in (1, 2, 3, 4, 5, 6, 8, 10, 14, 20):
                try:
                    t, f, ta = run(nsys, f"{R},{NT},{c}")
                except Exception as ex:  # noqa: BLE001
                    continue
                res.append((ta, t, f, R, NT, c))
    res.sort()
    for ta, t, f, R, NT, c in res[:8]:
        print(f"   R={R} NT={NT} c={c}: application {ta:.1f} us, kernel {t:.1f} us frac {f:.3f}", flush=True)
