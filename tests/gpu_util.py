"""Helpers for the -m gpu parity tests (CUDA path vs the fp64 oracle)."""
import numpy as np
import pytest
import torch

requires_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def to_np(t):
    return t.detach().cpu().numpy()


def soa_to_aos(t):
    return np.ascontiguousarray(to_np(t).T)
