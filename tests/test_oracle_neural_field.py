"""Pins of oracle.neural_field (NEXT-4) against properties that do not
reuse its formulas: trilinear interpolation reproduces linear fields exactly and returns
vertex values at vertices, PE values at known points, the explicit backward pass against
central finite differences of the loss (fp64, every parameter block), the MSE gradient,
and Adam's first step in closed form."""
import math

import numpy as np
import pytest
import torch

import nat_inputs as I
from oracle import neural_field as NF


def _params(n_v, n_out, seed, dtype=torch.float64, grid_scale=1e-4):
    shapes = [s for _, s in NF.param_layout(n_v, n_out)]
    flat = I.nf_init_params(shapes, seed, grid_scale=grid_scale)
    return torch.from_numpy(flat).to(dtype)


def test_dense_tables_and_vertex_index():
    for l in range(NF.LEVELS):
        n = NF.level_res(l) + 1
        assert NF.level_size(l) == n ** 3            # every level fits 2^19 rows: dense
        idx = NF.vertex_index(l, torch.tensor([0, n - 1, 3]), torch.tensor([0, n - 1, 2]), torch.tensor([0, n - 1, 1]))
        assert idx.tolist() == [0, n ** 3 - 1, 3 + n * (2 + n * 1)]


def test_trilinear_reproduces_linear_fields_and_vertex_values():
    """Grid features set to a linear function of the vertex position: the encoding at any x
    equals the function at x (trilinear interpolation is exact for affine fields)."""
    torch.manual_seed(0)
    a = torch.tensor([[0.3, -1.2, 2.0, 0.5], [1.0, 0.25, -0.7, 2.0], [-0.4, 0.9, 0.1, -1.5]], dtype=torch.float64)
    b = torch.tensor([0.1, -0.2, 0.3, 0.05], dtype=torch.float64)
    grids = []
    for l in range(NF.LEVELS):
        n = NF.level_res(l)
        ii = torch.arange(n + 1, dtype=torch.float64) / n
        K, J, Ii = torch.meshgrid(ii, ii, ii, indexing="ij")
        pos = torch.stack([Ii.reshape(-1), J.reshape(-1), K.reshape(-1)], 1)   # row = i + (n+1)(j + (n+1)k)
        grids.append(pos @ a + b)
    x = torch.rand(500, 3, dtype=torch.float64)
    x[0] = torch.tensor([1.0, 1.0, 1.0])
    x[1] = torch.tensor([0.0, 0.0, 0.0])
    feats, _, ws = NF.grid_encode(x, grids)
    expect = x @ a + b
    for l in range(NF.LEVELS):
        assert torch.allclose(feats[:, 4 * l:4 * l + 4], expect, atol=1e-13)
        assert torch.allclose(ws[l].sum(1), torch.ones(500, dtype=torch.float64), atol=1e-14)
    # at a lattice vertex the encoding is that vertex's feature vector
    n = NF.level_res(3)
    xv = torch.tensor([[5 / n, 17 / n, 63 / n]], dtype=torch.float64)
    fv, _, _ = NF.grid_encode(xv, grids)
    assert torch.allclose(fv[0, 12:16], grids[3][5 + (n + 1) * (17 + (n + 1) * 63)], atol=1e-14)


def test_positional_encoding_values():
    v = torch.tensor([[0.25, 0.0]], dtype=torch.float64)
    pe = NF.positional(v)
    assert pe.shape == (1, 24)
    # v = 1/4: sin(2^k pi / 4) = sqrt(2)/2, 1, 0, 0, ... ; cos: sqrt(2)/2, 0, -1, 1, 1, 1
    s = [math.sqrt(0.5), 1.0, 0.0, 0.0, 0.0, 0.0]
    c = [math.sqrt(0.5), 0.0, -1.0, 1.0, 1.0, 1.0]
    assert torch.allclose(pe[0, 0:12:2], torch.tensor(s, dtype=torch.float64), atol=1e-15)
    assert torch.allclose(pe[0, 1:12:2], torch.tensor(c, dtype=torch.float64), atol=1e-15)
    assert torch.allclose(pe[0, 12:24], torch.tensor([0.0, 1.0] * 6, dtype=torch.float64))


def test_backward_matches_finite_differences():
    """fp64, no bf16 rounding: d loss / d theta from the explicit backward pass against
    central differences, sampled entries of every parameter block."""
    n_v, n_out, B = 3, 8, 24
    flat = _params(n_v, n_out, 7, grid_scale=0.5)
    rng = np.random.default_rng(1)
    inputs = torch.from_numpy(rng.random((B, 3 + n_v)))
    targets = torch.from_numpy(rng.random((B, n_out)))
    Y, cache = NF.forward(flat, inputs, n_out, use_bf16=False)
    L, dY = NF.loss_grad(Y, targets)
    g = NF.backward(flat, inputs, n_out, dY, cache, use_bf16=False)
    off = 0
    h = 1e-6
    for name, shp in NF.param_layout(n_v, n_out):
        n = math.prod(shp)
        blk = g[off:off + n]
        # entries the batch touches (grid rows of the visited voxels) and random others
        cand = torch.nonzero(blk).flatten()
        pick = cand[torch.randperm(len(cand), generator=torch.Generator().manual_seed(3))[:4]] if len(cand) else []
        for e in list(pick):
            i = off + int(e)
            fp, fm = flat.clone(), flat.clone()
            fp[i] += h
            fm[i] -= h
            lp = NF.loss_grad(NF.forward(fp, inputs, n_out, use_bf16=False)[0], targets)[0]
            lm = NF.loss_grad(NF.forward(fm, inputs, n_out, use_bf16=False)[0], targets)[0]
            fd = float((lp - lm) / (2 * h))
            assert abs(fd - float(g[i])) <= 1e-6 * max(1.0, abs(fd)) + 1e-9, (name, int(e), fd, float(g[i]))
        assert len(cand) > 0, name
        off += n


def test_mse_gradient_and_adam_first_step():
    Y = torch.tensor([[1.0, 2.0], [3.0, 5.0]], dtype=torch.float64)
    T = torch.tensor([[0.0, 2.0], [4.0, 1.0]], dtype=torch.float64)
    L, dY = NF.loss_grad(Y, T)
    assert float(L) == (1 + 0 + 1 + 16) / 4
    assert torch.equal(dY, torch.tensor([[0.5, 0.0], [-0.5, 2.0]], dtype=torch.float64))
    # Adam's first bias-corrected step is -lr * g / (|g| + eps)
    p = torch.tensor([1.0, -2.0, 0.5], dtype=torch.float64)
    g = torch.tensor([0.3, -4.0, 0.0], dtype=torch.float64)
    m, v = torch.zeros(3, dtype=torch.float64), torch.zeros(3, dtype=torch.float64)
    p0 = p.clone()
    NF.adam(p, g, m, v, 1, 1e-3)
    assert torch.allclose(p - p0, -1e-3 * g / (g.abs() + 1e-8), atol=1e-15)


def test_bf16_rounding_is_where_the_gpu_rounds():
    """The bf16 network differs from the fp32 one by bf16-size relative errors only."""
    n_v, n_out, B = 3, 8, 64
    flat = _params(n_v, n_out, 5, dtype=torch.float32, grid_scale=0.5)
    inputs = torch.from_numpy(np.random.default_rng(2).random((B, 3 + n_v))).float()
    y16, _ = NF.forward(flat, inputs, n_out, use_bf16=True)
    y32, _ = NF.forward(flat, inputs, n_out, use_bf16=False)
    rel = float(torch.linalg.norm(y16 - y32) / torch.linalg.norm(y32))
    assert 1e-5 < rel < 3e-2
