"""Diagnose: sequential steps after overlapped ones (phase times and a kernel timeline)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2506_06190_b200 import nat  # noqa: E402

torch.cuda.set_device(0)
nat.lib()
step = bench.Step(nat, torch, 0, 1, None, bench.load_host())
for ov in (True, True, True, True, False, False):
    step.ev = {}
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step.run(overlap=ov)
    e1.record()
    torch.cuda.synchronize()
    print(ov, round(e0.elapsed_time(e1), 3), {k: round(v, 3) for k, v in step.phase_ms().items()})
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step.run(overlap=False)
    torch.cuda.synchronize()
recs = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
              if e.device_type == torch.autograd.DeviceType.CUDA)
t0 = recs[0][0]
last = t0
for s, en, nm in recs[:80]:
    print(f"{s - t0:10.1f} {en - s:9.1f} {max(0, s - last):8.1f} {nm[:90]}")
    last = max(last, en)
