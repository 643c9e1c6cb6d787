import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2506_06190_b200 import nat
S, P, nm = 61440, 32768, 3
rng = np.random.default_rng(0)
y = rng.normal(size=(3, S)); y /= np.linalg.norm(y, axis=0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
x = T(y[:, :P] * 2.0)
src = nat.Sources(T(y), T(y), T(np.full(S, 1e-3)), T(np.ones((nm, S), complex)), T(np.zeros((nm, S), complex)))
plan = nat.RadiatePlan(S, nm, P, "fp32")
out = nat.nat_radiate_field(src, [1.0, 2.0, 3.0], x, "fp32", plan=plan)
torch.cuda.synchronize(); print("ok", out.abs().max().item())
