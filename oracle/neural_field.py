"""NEXT-4: the NAT neural acoustic transfer field (§3.2-3.3, l.120-162) — oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain PyTorch on the CPU, written
from the paper step by step (reading R-nf):

  Phi(theta, phi, r, v) = MLP[ G(theta, phi, r) ; P(v) ]                    (l.131-136)
  G  = the multi-resolution feature grid (l.141-152): L = 4 levels of 3D lattices over the
       normalised (theta, phi, r) in [0, 1]^3, resolutions N_l = 8 * 2^l (8 .. 64, l.158),
       F = 4 features per lattice vertex, trilinear interpolation of the 8 vertices of the
       voxel enclosing x, levels concatenated (16 features).  The lattices ((N+1)^3 <= 2^19
       vertices each) are stored densely; the hash of instant-NGP (l.152) applies only above
       `table` entries and is implemented for completeness.
  P  = NeRF positional encoding of each condition variable v_d in [0, 1] (l.137, l.158):
       sin(2^k pi v_d), cos(2^k pi v_d), k = 0..5.
  MLP = 4 hidden layers of 128 neurons, ReLU after each layer except the last (l.156);
       the input (16 + 12 n_v features) is zero-padded to 64 columns; n_out outputs (the
       |p| of each mode, l.156).
  loss = mean squared error over the batch and the outputs (l.124).
  Adam (l.158), default moments (beta1, beta2, eps) = (0.9, 0.999, 1e-8).

Precision: the GPU runs every layer product on bf16 tensor cores with fp32 accumulation;
this oracle rounds the same operands to bf16 at the same places (activations and weights
entering each product, forward and backward) and keeps everything else in fp32, so the
two differ only by summation order.  `bf16=False` gives the exact fp32/fp64 network the
pins use (finite differences).

Pinned by tests/test_oracle_neural_field.py: trilinear reproduction of linear fields,
vertex values, the dense index, PE values, the backward pass against central finite
differences (fp64, every parameter block), the MSE gradient and Adam's first step in
closed form.
"""
import math

import torch

LEVELS, FEATURES, BASE_RES, TABLE = 4, 4, 8, 1 << 19
PE_FREQS = 6
IN_PAD, HIDDEN, N_HIDDEN = 64, 128, 4
PRIMES = (1, 2654435761, 805459861)


def level_res(l):
    return BASE_RES * (2 ** l)


def level_size(l):
    n = level_res(l) + 1
    return min(n ** 3, TABLE)


def vertex_index(l, i, j, k):
    """Table row of lattice vertex (i, j, k) on level l: dense i + (N+1)(j + (N+1) k) when
    the lattice fits the table, else the instant-NGP spatial hash."""
    n = level_res(l) + 1
    if n ** 3 <= TABLE:
        return i + n * (j + n * k)
    h = (i * PRIMES[0]) ^ (j * PRIMES[1]) ^ (k * PRIMES[2])
    return h % TABLE


def param_layout(n_v, n_out):
    """[(name, shape)] of the parameter vector (grid tables, then per layer W [out][in], b)."""
    shapes = [(f"grid{l}", (level_size(l), FEATURES)) for l in range(LEVELS)]
    dims = [IN_PAD] + [HIDDEN] * N_HIDDEN + [n_out]
    for q in range(len(dims) - 1):
        shapes.append((f"W{q}", (dims[q + 1], dims[q])))
        shapes.append((f"b{q}", (dims[q + 1],)))
    return shapes


def unpack(flat, n_v, n_out):
    out, o = {}, 0
    for name, shp in param_layout(n_v, n_out):
        n = math.prod(shp)
        out[name] = flat[o:o + n].view(shp)
        o += n
    return out


def bf16(t, on=True):
    return t.to(torch.bfloat16).to(t.dtype) if on else t


def grid_encode(x, grids):
    """x [B][3] in [0, 1]; returns (features [B][L*F], corner rows [L][B][8], weights [L][B][8])."""
    feats, rows_all, w_all = [], [], []
    for l in range(LEVELS):
        n = level_res(l)
        p = x * n
        i0 = torch.clamp(torch.floor(p), 0, n - 1).to(torch.int64)
        f = p - i0.to(p.dtype)
        rows, ws = [], []
        acc = torch.zeros(x.shape[0], FEATURES, dtype=x.dtype)
        for c in range(8):
            dx, dy, dz = c & 1, (c >> 1) & 1, (c >> 2) & 1
            wx = f[:, 0] if dx else 1 - f[:, 0]
            wy = f[:, 1] if dy else 1 - f[:, 1]
            wz = f[:, 2] if dz else 1 - f[:, 2]
            w = (wx * wy) * wz
            r = vertex_index(l, i0[:, 0] + dx, i0[:, 1] + dy, i0[:, 2] + dz)
            acc = acc + w[:, None] * grids[l][r]
            rows.append(r)
            ws.append(w)
        feats.append(acc)
        rows_all.append(torch.stack(rows, 1))
        w_all.append(torch.stack(ws, 1))
    return torch.cat(feats, 1), rows_all, w_all


def positional(v):
    """v [B][n_v] in [0, 1] -> [B][12 n_v]: per dimension d, per k: sin(2^k pi v_d), cos(2^k pi v_d)."""
    cols = []
    for d in range(v.shape[1]):
        for k in range(PE_FREQS):
            a = (2.0 ** k) * math.pi * v[:, d]
            cols += [torch.sin(a), torch.cos(a)]
    return torch.stack(cols, 1)


def encode(inputs, P):
    """inputs [B][3 + n_v] = (theta^, phi^, r^, v) -> X [B][64] (zero padded) + grid cache."""
    x, v = inputs[:, :3], inputs[:, 3:]
    g, rows, ws = grid_encode(x, [P[f"grid{l}"] for l in range(LEVELS)])
    pe = positional(v)
    X = torch.zeros(inputs.shape[0], IN_PAD, dtype=inputs.dtype)
    X[:, : g.shape[1]] = g
    X[:, g.shape[1]: g.shape[1] + pe.shape[1]] = pe
    return X, (rows, ws)


def forward(flat, inputs, n_out, use_bf16=True):
    """Returns (Y [B][n_out], cache)."""
    n_v = inputs.shape[1] - 3
    P = unpack(flat, n_v, n_out)
    X, gc = encode(inputs, P)
    acts = [X]
    h = X
    for q in range(N_HIDDEN + 1):
        z = bf16(h, use_bf16) @ bf16(P[f"W{q}"], use_bf16).T + P[f"b{q}"]
        h = torch.relu(z) if q < N_HIDDEN else z
        acts.append(h)
    return h, (P, acts, gc)


def loss_grad(Y, T):
    """MSE (l.124) and its gradient with respect to Y."""
    d = Y - T
    return (d * d).mean(), 2.0 * d / d.numel()


def backward(flat, inputs, n_out, dY, cache, use_bf16=True):
    """Gradient of sum(dY * Y) with respect to every parameter (same layout as flat)."""
    P, acts, (rows, ws) = cache
    n_v = inputs.shape[1] - 3
    G = {k: torch.zeros_like(v) for k, v in P.items()}
    d = dY
    for q in range(N_HIDDEN, -1, -1):
        h_in = acts[q]
        G[f"W{q}"] = bf16(d, use_bf16).T @ bf16(h_in, use_bf16)
        G[f"b{q}"] = d.sum(0)
        dh = bf16(d, use_bf16) @ bf16(P[f"W{q}"], use_bf16)
        d = dh * (h_in > 0).to(dh.dtype) if q > 0 else dh
    # d = dL/dX; the grid part scatters to the 8 corner vertices of each level
    for l in range(LEVELS):
        dg = d[:, l * FEATURES:(l + 1) * FEATURES]
        for c in range(8):
            G[f"grid{l}"].index_add_(0, rows[l][:, c], ws[l][:, c][:, None] * dg)
    return torch.cat([G[name].reshape(-1) for name, _ in param_layout(n_v, n_out)])


def adam(flat, grad, m, v, step, lr, b1=0.9, b2=0.999, eps=1e-8):
    """One Adam step (Kingma & Ba) in place; step counts from 1."""
    m.mul_(b1).add_((1 - b1) * grad)
    v.mul_(b2).add_((1 - b2) * grad * grad)
    mh = m / (1 - b1 ** step)
    vh = v / (1 - b2 ** step)
    flat.sub_(lr * mh / (torch.sqrt(vh) + eps))


def train_step(flat, m, v, step, lr, inputs, targets, n_out, use_bf16=True):
    """Forward, MSE, backward, Adam; returns the loss before the update."""
    Y, cache = forward(flat, inputs, n_out, use_bf16)
    L, dY = loss_grad(Y, targets)
    g = backward(flat, inputs, n_out, dY, cache, use_bf16)
    adam(flat, g, m, v, step, lr)
    return float(L)
