"""Times nat_radiate_field at given shapes for forced launch plans (NAT_RAD_PLAN)."""
import os
import subprocess
import sys

CODE = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2506_06190_b200 import nat
S, P, nm, self_mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rng = np.random.default_rng(0)
y = rng.normal(size=(3, S)); y /= np.linalg.norm(y, axis=0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
x = T(y) if self_mode else T(y * 2.0)
src = nat.Sources(T(y), T(y), T(np.full(S, 1e-3)), T(np.ones((nm, S), complex)), T(np.zeros((nm, S), complex)))
ks = list(np.linspace(0.5, 8, nm))
plan = nat.RadiatePlan(S, nm, P, "fp32")
out = nat.nat_radiate_field(src, ks, x, "fp32", plan=plan)
for _ in range(3): nat.nat_radiate_field(src, ks, x, "fp32", out=out, plan=plan)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): nat.nat_radiate_field(src, ks, x, "fp32", out=out, plan=plan)
e1.record(); torch.cuda.synchronize()
print(e0.elapsed_time(e1) / 20 * 1e3)
'''

def run(shape, plan):
    env = dict(os.environ)
    if plan:
        env["NAT_RAD_PLAN"] = plan
    else:
        env.pop("NAT_RAD_PLAN", None)
    r = subprocess.run([sys.executable, "-c", CODE] + [str(v) for v in shape], env=env, capture_output=True, text=True)
    return float(r.stdout.strip().split()[-1]) if r.returncode == 0 else float("nan")

for shape in [(10000, 10000, 1, 0), (10000, 10000, 3, 0), (61440, 32768, 3, 0)]:
    pairs = shape[0] * shape[1] * shape[2]
    auto = run(shape, None)
    print(f"shape {shape}: auto {auto:.1f} us ({pairs / auto / 1e6 / 1.551:.1%} of R_pipe)", flush=True)
    res = []
    cs = [1, 2, 3, 4, 6, 8, 10, 14, 20] if shape[0] == 10000 else [8, 16, 24, 32, 40, 48, 60, 80]
    for R in (2, 4):
        for NT in (128, 256):
            for c in cs:
                t = run(shape, f"{R},{NT},{c}")
                res.append((t, R, NT, c))
    res.sort()
    for t, R, NT, c in res[:6]:
        print(f"   R={R} NT={NT} c={c}: {t:.1f} us ({pairs / t / 1e6 / 1.551:.1%})", flush=True)
