"""NEXT-4 (the NAT neural field) on the GPU: the tcgen05 tensor-core
product in every operand layout against torch, the forward pass and training steps
against oracle/neural_field.py (which rounds the same operands to bf16)."""
import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import rel_l2, requires_cuda, to_np
from oracle import neural_field as NF

pytestmark = [pytest.mark.gpu, requires_cuda]


def _nat():
    from paper_2506_06190_b200 import nat
    return nat


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (304, 64, 200), (1000, 16, 1024), (136, 32, 16)])
def test_tcgen05_gemm_layouts(a_mn, b_mn, M, N, K):
    nat = _nat()
    g = torch.Generator().manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16)
    ref = A.double() @ B.double().T           # exact products of the bf16 operands
    Ad = (A.T.contiguous() if a_mn else A).cuda()
    Bd = (B.T.contiguous() if b_mn else B).cuda()
    C = nat.nat_nf_gemm_bf16(Ad, Bd, a_mn, b_mn).cpu()
    assert rel_l2(C.numpy(), ref.numpy()) <= 1e-5  # fp32 accumulation over K <= 1024


def _case(n, n_v=3, n_out=8, seed=4):
    shapes = [s for _, s in NF.param_layout(n_v, n_out)]
    flat = I.nf_init_params(shapes, seed, grid_scale=0.05)
    x = I.nf_samples(n, n_v, seed + 1)
    t = np.random.default_rng(seed + 2).random((n, n_out)).astype(np.float32)
    return flat, x, t


def test_param_layout_matches_oracle():
    nat = _nat()
    for n_v, n_out in ((3, 8), (1, 1), (4, 16)):
        assert nat.NeuralField.param_count(n_v, n_out) == sum(int(np.prod(s)) for _, s in NF.param_layout(n_v, n_out))
        assert [tuple(s) for s in nat.NeuralField.param_shapes(n_v, n_out)] == \
            [tuple(s) for _, s in NF.param_layout(n_v, n_out)]


@pytest.mark.parametrize("n", [128, 1000, 8192])
def test_forward_parity(n):
    nat = _nat()
    flat, x, _ = _case(n)
    net = nat.NeuralField(3, 8, torch.from_numpy(flat).cuda(), n)
    y = to_np(net.forward(torch.from_numpy(x).cuda()))
    y_ref, _ = NF.forward(torch.from_numpy(flat), torch.from_numpy(x), 8, use_bf16=True)
    assert rel_l2(y, y_ref.numpy()) <= 2e-3


def test_train_steps_parity():
    """Three Adam steps: the loss of every step, the first step's gradient per parameter
    block, and the parameters after three steps against the oracle on the same batch."""
    nat = _nat()
    n, lr = 4096, 1e-3
    flat, x, t = _case(n)
    net = nat.NeuralField(3, 8, torch.from_numpy(flat).cuda(), n)
    xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    ref = torch.from_numpy(flat).clone()
    m, v = torch.zeros_like(ref), torch.zeros_like(ref)
    xr, tr = torch.from_numpy(x), torch.from_numpy(t)
    grad = torch.zeros_like(net.params)
    for step in range(1, 4):
        Y, cache = NF.forward(ref, xr, 8)
        L, dY = NF.loss_grad(Y, tr)
        g_ref = NF.backward(ref, xr, 8, dY, cache)
        loss = float(net.train_step(xd, td, lr, grad_out=grad if step == 1 else None).item())
        assert abs(loss - float(L)) <= 1e-3 * float(L)
        if step == 1:
            gg = grad.cpu()
            off = 0
            for name, shp in NF.param_layout(3, 8):
                k = int(np.prod(shp))
                a, b = gg[off:off + k].numpy(), g_ref[off:off + k].numpy()
                assert rel_l2(a, b) <= 2e-2, name
                off += k
        NF.adam(ref, g_ref, m, v, step, lr)
    # Adam's normalised step m/sqrt(v) turns the rounding noise of near-zero gradients into
    # steps of size ~lr: the parameters agree to ~1e-3 while the loss agrees to 1e-3 per step
    assert rel_l2(net.params.cpu().numpy(), ref.numpy()) <= 1e-3


def test_training_reduces_the_loss():
    nat = _nat()
    n = 16384
    flat, x, _ = _case(n, seed=9)
    xt = torch.from_numpy(x).cuda()
    # a smooth target field of (theta, phi, r, v): the network must fit it
    tgt = torch.stack([torch.sin(3 * xt[:, 0] + q) * torch.cos(2 * xt[:, 1]) * (1 + xt[:, 3 + q % 3]) for q in range(8)], 1)
    net = nat.NeuralField(3, 8, torch.from_numpy(flat).cuda(), n)
    first = None
    for _ in range(200):
        L = float(net.train_step(xt, tgt.contiguous(), 1e-3).item())
        first = L if first is None else first
    assert L < 0.1 * first
