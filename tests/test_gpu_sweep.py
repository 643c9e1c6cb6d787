"""The C4 sweep job end to end on the GPU (2 geometries, 8^3 listeners): result files,
manifest, resume (a rerun does no work), and the stored fields against a direct
nat_radiate_field of the same geometry."""
import json
import os

import numpy as np
import pytest

from gpu_util import requires_cuda

pytestmark = [pytest.mark.gpu, requires_cuda]


def test_sweep_files_resume_and_manifest(tmp_path):
    from paper_2506_06190_b200 import sweep
    d = str(tmp_path)
    logs = []
    sweep.run(d, n_geo=2, grid=8, workers=2, log=logs.append)
    assert sweep.todo(d, [0, 1]) == []
    man = sweep.write_manifest(d, 2, {"config": "C4 test"})
    for gi in (0, 1):
        rec = man["records"][str(gi)]
        assert len(rec["iters"]) == 64 and rec["field_shape"] == [64, 512]
        assert all(0 < it <= 200 for it in rec["iters"])
        f = np.load(sweep.geo_file(d, gi, "npy"))
        assert np.all(np.isfinite(f)) and np.abs(f).max() > 0
    logs.clear()
    sweep.run(d, n_geo=2, grid=8, workers=2, log=logs.append)      # resume: nothing left
    assert "2 already done" in logs[0] and not any("geometry" in l and ": " in l and " s," in l for l in logs)
    # geometry 1's field equals a direct computation of the same geometry (c64 storage)
    import torch
    from paper_2506_06190_b200 import nat
    bufs = {"mc": nat.McPlan(sweep.M_SAMPLES, 64, "fp32", 200, "cuda"),
            "rad": nat.RadiatePlan(sweep.M_SAMPLES, 64, 512, "fp32", "cuda")}
    out, rec = sweep.run_geometry(nat, torch, 1, 8, bufs)
    f1 = np.load(sweep.geo_file(d, 1, "npy"))
    ref = out.cpu().numpy()
    assert np.linalg.norm(f1 - ref) / np.linalg.norm(ref) < 1e-6
    assert json.load(open(sweep.geo_file(d, 1, "json")))["iters"] == rec["iters"]
