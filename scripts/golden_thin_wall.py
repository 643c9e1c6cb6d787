"""Writes tests/golden/thin_wall.txt: the ORACLE's relative L2 error of the radiated field
for the thin-wall interior point source (SURVEY §8(d) C3 acceptance; P:398's analytic
point-source idea) on the bowl at 832 and 3,200 triangles.  Calls only oracle/ (and the
input generators); the GPU test compares the CUDA path's error on the same problem with it.

    python scripts/golden_thin_wall.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_oracle_bem import _thin_wall_case  # noqa: E402  (oracle-only helper)

rows = [(32, 6), (64, 12)]
with open(os.path.join(ROOT, "tests", "golden", "thin_wall.txt"), "w") as f:
    f.write("# Thin-wall interior point source x_s = (0, 0, -0.95), k = 2, bowl(n_az, n_psi, 2): relative L2\n"
            "# error of the oracle's radiated field against G(x, x_s) at the 8x8x4 shell grid (oracle: dense\n"
            "# P0 collocation, GMRES tol 1e-10).  Written by scripts/golden_thin_wall.py (oracle only).\n"
            "# columns: n_az n_psi n_tri rel_l2\n")
    for n_az, n_psi in rows:
        e = _thin_wall_case(n_az, n_psi)
        n_tri = n_az * (2 * (2 * n_psi - 1) + 4)
        f.write(f"{n_az} {n_psi} {n_tri} {e:.15e}\n")
        print(n_az, n_psi, n_tri, e, flush=True)
