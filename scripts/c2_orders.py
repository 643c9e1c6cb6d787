"""C2 step time under each NAT_BENCH_ORDER (interleave / asm_first / multi), 1 GPU, 3 reps each."""
import os
import sys

import torch

sys.path.insert(0, ".")
import bench_secondary as S
from paper_2506_06190_b200 import nat

nat.lib()
for rep in range(3):
    for order in ("interleave", "asm_first", "multi"):
        os.environ["NAT_BENCH_ORDER"] = order
        r = S.run_c2(nat, torch, 0, 1, None, 5, lambda: None, lambda a, b: (a, b))
        print(f"{order:10s} {r['ms_per_step']:.2f} ms  {r['value']:.0f} Gpair-evals/s  iters {r['gmres_iters']}", flush=True)
