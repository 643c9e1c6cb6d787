"""NEXT-4 training step timing (bench_secondary.run_nf) plus the per-product kernel-timer split."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import bench_secondary as S
from paper_2506_06190_b200 import nat

nat.lib()
pk = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else None
for _ in range(2):
    r = S.run_nf(nat, torch, 10, peaks=pk)
    g = r["gemm"]
    print(f"step {r['ms_per_step']:.3f} ms, gemm {g['gemm_ms_per_step']:.3f} ms, {g['achieved']:.0f} GB/s "
          f"({g['frac']:.3f} of HBM), tensor view {g['tensor_view']['achieved']:.1f} TFLOP/s, loss {r['loss']:.4f}",
          flush=True)
