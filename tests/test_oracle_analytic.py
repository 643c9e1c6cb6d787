"""Pin of oracle.analytic against the values SPEC prints (tests/golden/sphere_values.txt)."""
from oracle import analytic

def test_pulsating_sphere_matches_spec_printed_values():
    """tests/golden/sphere_values.txt: |p(r)| printed by SPEC S:119-123 for a = g = k = 1."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "sphere_values.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    assert len(rows) == 2
    for r, ap, tol in rows:
        assert abs(abs(analytic.pulsating_sphere(float(r), 1.0)) - float(ap)) <= float(tol)
