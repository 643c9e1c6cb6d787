import torch, time, sys
sys.path.insert(0, '.')
from paper_2506_06190_b200 import nat
import numpy as np
for rows, n in ((1024, 199692), (24962, 199692 // 8 * 8), (20480, 20480)):
    A = torch.randn(rows, n, dtype=torch.complex128, device="cuda")
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    y = torch.empty(rows, dtype=torch.complex128, device="cuda")
    nat.nat_bem_matvec(A, x, n=n, out=y)
    torch.cuda.synchronize()
    ref = (A @ x)
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        nat.nat_bem_matvec(A, x, n=n, out=y)
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 5 * 1e-3
    print(rows, n, "err", err, "GB/s", rows * n * 16 / t / 1e9)
    del A
