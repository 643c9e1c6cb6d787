"""Pins of oracle.philox against the Random123 known-answer vectors."""
import numpy as np

from conftest import load_golden
from oracle import philox


def test_philox_kat():
    for row in load_golden("philox_kat.txt"):
        vals = [int(v, 16) for v in row]
        ctr, key, out = vals[:4], vals[4:6], vals[6:]
        got = philox.philox4x32_10(np.array([ctr], dtype=np.uint64), key)[0]
        assert [int(v) for v in got] == out


def test_uniforms_open_interval_and_exact():
    u = philox.uniforms(np.arange(1000), 0, 3, 20250606)
    assert np.all(u > 0) and np.all(u < 1)
    o = np.round(u * 2.0 ** 32 - 0.5)
    assert np.array_equal((o + 0.5) * 2.0 ** -32, u)
