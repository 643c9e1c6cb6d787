"""Diagnose the pipelined sweep: NaN / mismatch per geometry under worker / serial variants."""
import sys

import torch

sys.path.insert(0, ".")
import bench
from paper_2506_06190_b200 import nat

nat.lib()
sweep = bench.Sweep(nat, torch, 0, 1, 2, n_geo=64, e2e=False)
ids = [0, 9, 33, 63]
for nw, serial in ((1, True), (1, False), (2, True), (2, False), (2, False)):
    keep = {}
    sweep.run(geo_ids=ids, keep=keep, n_workers=nw, serial=serial)
    torch.cuda.synchronize()
    print(nw, serial, {gi: int(torch.isnan(v).sum()) for gi, v in keep.items()}, flush=True)
