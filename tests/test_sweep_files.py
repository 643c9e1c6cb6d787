"""The C4 sweep's result files, manifest and resume bookkeeping (paper_2506_06190_b200/
sweep.py; SURVEY §5 checkpoint/resume) — host logic only, no GPU."""
import json
import os

import numpy as np
import pytest

from paper_2506_06190_b200 import sweep


def _rec(gi):
    return {"geometry": gi, "iters": [3, 4], "converged": [True, True]}


def test_geometry_done_only_after_both_files(tmp_path):
    d = str(tmp_path)
    assert not sweep.is_done(d, 0)
    f = (np.arange(6) + 1j).reshape(2, 3)
    sweep.save_geometry(d, 0, f, _rec(0))
    assert sweep.is_done(d, 0)
    rec = json.load(open(sweep.geo_file(d, 0, "json")))
    assert rec["field_shape"] == [2, 3] and rec["field_dtype"] == "complex64"
    assert np.array_equal(np.load(sweep.geo_file(d, 0, "npy")), f.astype(np.complex64))
    # a truncated field file (interrupted copy) is not done
    with open(sweep.geo_file(d, 0, "npy"), "r+b") as fh:
        fh.truncate(10)
    assert not sweep.is_done(d, 0)
    # a field without its record (interrupted before the .json) is not done
    sweep.save_geometry(d, 1, f, _rec(1))
    os.remove(sweep.geo_file(d, 1, "json"))
    assert not sweep.is_done(d, 1)
    assert not any(n.endswith(".tmp") for n in os.listdir(d))


def test_resume_list_and_manifest_written_last(tmp_path):
    d = str(tmp_path)
    f = np.zeros((2, 3), complex)
    for gi in (0, 2):
        sweep.save_geometry(d, gi, f, _rec(gi))
    assert sweep.todo(d, [0, 1, 2, 3]) == [1, 3]
    with pytest.raises(RuntimeError, match="geometry 1 missing"):
        sweep.write_manifest(d, 4, {})
    assert not os.path.exists(os.path.join(d, "manifest.json"))
    for gi in (1, 3):
        sweep.save_geometry(d, gi, f, dict(_rec(gi), converged=[True, gi != 3]))
    man = sweep.write_manifest(d, 4, {"config": "C4"})
    assert man["geometries"] == 4 and man["all_converged"] is False
    assert json.load(open(os.path.join(d, "manifest.json")))["records"]["3"]["converged"] == [True, False]
