"""Probe: time the sum of 16 split-K partial planes [16][64 x 2048] c128 (33.5 MB) with
torch, plane stride a power of two vs padded (L2 hashing check for mc_finish)."""
import torch

n = 64 * 2048
for pad in (0, 64, 1024):
    base = torch.randn(16, n + pad, dtype=torch.complex128, device="cuda")
    part = base[:, :n]
    out = torch.empty(n, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        torch.sum(part, 0, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        torch.sum(part, 0, out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 10
    print(f"pad {pad}: {us:.2f} us per sum, {16 * n * 16 / us / 1e6:.2f} TB/s")
