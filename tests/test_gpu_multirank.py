"""The library's world > 1 code path, executed: 2 and 4 ranks (processes) on the one GPU
of this box, all-gathers through the host-staged communicator (nat_comm_create_host over
a gloo group: no kernel waits on another rank).  SURVEY §8(e) / §4: the row-sharded dense
solve (stored matrix and matrix-free) and the row-sharded MC solve must return the SAME
iterate on every rank and for every rank count — bit for bit (fixed-order reductions that
do not depend on the row split; the MC pair kernels choose their launch shape for the full
operator, `RadInput::plan_lis`)."""
import os
import socket

import numpy as np
import pytest
import torch

import nat_inputs as I
from gpu_util import requires_cuda

pytestmark = [pytest.mark.gpu, requires_cuda]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases(nat, comm, rank, world):
    """Runs every sharded solve; returns numpy copies of the replicated solutions."""
    out = {}
    # dense BEM, stored matrix, fp64 (tol 1e-12) and fp32 (tol 1e-6)
    m = I.icosphere(3)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
    r0, r1 = nat.row_range(m.n_tri, rank, world)
    near = nat.nat_bem_near_list(mesh, geo, r0, r1)
    for prec, tol in (("fp64", 1e-12), ("fp32", 1e-6)):
        A, b = nat.nat_bem_assemble(mesh, geo, near, 3.0, g, prec=prec)
        x, info = nat.nat_bem_solve(A, b[0], m.n_tri, r0, comm, tol=tol)
        out[f"bem_{prec}"] = (x.cpu().numpy(), info["iters"])
    # matrix-free dense operator (NEXT-3b), fp64
    op, rhs = nat.nat_bem_mf_prepare(mesh, geo, near, 3.0, g, prec="fp64")
    x, info = nat.nat_bem_mf_solve(op, rhs[0], comm, tol=1e-12)
    out["mf_fp64"] = (x.cpu().numpy(), info["iters"])
    # row-sharded BEM-MC, 3 wavenumbers sharing one sample set, fp32 and fp64
    bm = I.bowl(32, 8, 2)
    bmesh = nat.Mesh.from_numpy(bm.v, bm.t)
    bgeo = nat.nat_mesh_prepare(bmesh)
    gt = torch.from_numpy(I.neumann_harmonics(bm, 3)).cuda()
    for prec, tol in (("fp32", 1e-6), ("fp64", 1e-12)):
        _, _, p, infos = nat.nat_mc_surface_pressure_sharded(bmesh, bgeo, [0.5, 2.0, 4.5], gt, 701, comm, seed=3,
                                                             prec=prec, tol=tol)
        out[f"mc_{prec}"] = (p.cpu().numpy(), [i["iters"] for i in infos])
    torch.cuda.synchronize()
    return out


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2506_06190_b200 import nat
    comm = nat.Comm.host()
    try:
        res = _cases(nat, comm, rank, world)
        q.put((rank, res))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, repr(ex)))
    finally:
        comm.close()
        dist.destroy_process_group()


def _run(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    return res


@pytest.fixture(scope="module")
def world1():
    from paper_2506_06190_b200 import nat
    return _cases(nat, None, 0, 1)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_solves_bit_identical_across_ranks_and_world_sizes(world, world1):
    res = _run(world)
    for key, (ref, it_ref) in world1.items():
        for r in range(world):
            x, it = res[r][key]
            assert it == it_ref, (key, r, it, it_ref)
            assert np.array_equal(x, ref), (key, r, float(np.max(np.abs(x - ref))))


def test_host_comm_rejects_an_empty_rank():
    """M = 5 samples on 4 ranks: the last rank would own no rows — every rank fails the
    same check before any collective (no rank hangs); the callback is never called."""
    from paper_2506_06190_b200 import nat
    h = nat.Comm(0, 4, _host_fn=lambda *a: 1)
    bm = I.bowl(16, 4, 2)
    mesh = nat.Mesh.from_numpy(bm.v, bm.t)
    geo = nat.nat_mesh_prepare(mesh)
    g = torch.ones(1, bm.n_tri, dtype=torch.complex128, device="cuda")
    with pytest.raises(nat.NatError, match="owns no sample rows"):
        nat.nat_mc_surface_pressure_sharded(mesh, geo, [1.0], g, 5, h)
    h.close()
