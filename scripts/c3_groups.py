"""C3 secondary line (one MC call of 32 systems, M = 4096, + 32-mode radiation) under
solve groups 1 / 2 / 4."""
import sys

import torch

sys.path.insert(0, ".")
import bench_secondary as S
from paper_2506_06190_b200 import nat

nat.lib()
for G in (1, 2, 4, 1, 2):
    nat.nat_mc_set_groups(G)
    r = S.run_c3(nat, torch, 0, 1, 5, torch.cuda.synchronize, lambda a, b: (a, b))
    print(f"G={G}: {r['ms_per_step']:.2f} ms, {r['value']:.0f} Gpair-evals/s", flush=True)
