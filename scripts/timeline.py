"""GPU timeline of one bench step (torch.profiler / CUPTI kernel + memcpy records):
per-phase busy time vs span and the largest idle gaps, to find host-sync bubbles.

    python scripts/timeline.py > gpurun_out/timeline.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2506_06190_b200 import nat  # noqa: E402


def main():
    torch.cuda.set_device(0)
    nat.lib()
    host = bench.load_host()
    step = bench.Step(nat, torch, 0, 1, None, host)
    for _ in range(3):
        step.run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step.run()
        torch.cuda.synchronize()
    recs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            recs.append((e.time_range.start, e.time_range.end, e.name))
    recs.sort()
    t0 = recs[0][0]
    busy, last_end = 0.0, t0
    gaps = []
    rows = []
    for s, en, nm in recs:
        gap = max(0.0, s - last_end)
        if gap > 0:
            gaps.append((gap, s - t0, nm))
        busy += max(0.0, en - max(s, last_end))
        last_end = max(last_end, en)
        rows.append((s - t0, en - s, gap, nm))
    span = last_end - t0
    print(f"span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us, records {len(recs)}")
    gaps.sort(reverse=True)
    print("largest gaps (us, at, next kernel):")
    for g, at, nm in gaps[:40]:
        print(f"  {g:8.1f} {at:10.1f}  {nm[:90]}")
    # idle attributed to the kernel that follows the gap, summed by name
    agg = {}
    for g, at, nm in gaps:
        key = nm.split("(")[0][:70]
        a = agg.setdefault(key, [0.0, 0])
        a[0] += g
        a[1] += 1
    print("idle before kernel, summed:")
    for k, (g, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
        print(f"  {g:9.1f} us {c:5d}x  {k}")
    print("chronological:")
    for at, d, g, nm in rows:
        print(f"{at:10.1f} {d:9.1f} {g:8.1f}  {nm[:100]}")


if __name__ == "__main__":
    main()
