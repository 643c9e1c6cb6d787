"""The N > 1 host-side path on CPU, world_size = 2 over gloo (no GPU):

* the 128-byte NCCL unique-id broadcast protocol of nat.Comm;
* the row ownership the library enforces (rows_per_rank = ceil(n / world)) and the
  bench's listener / MC-wavenumber sharding tile their index sets exactly;
* the row-sharded GMRES protocol (local rows -> all-gather of the iterate -> replicated
  Arnoldi) emulated with the oracle's rows reproduces the single-process solution, for
  the dense BEM and for the row-sharded BEM-MC system (identical Philox samples
  regenerated on every rank);
* the bench's max-over-ranks timing reduction and sum-over-ranks work reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as ex:  # pragma: no cover
        q.put((rank, ex))
    finally:
        dist.destroy_process_group()


def _run(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, fn, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def _uid_fn(rank, world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2506_06190_b200.nat import Comm
    return Comm.broadcast_unique_id(make_id=lambda: bytes(range(128)))


def test_unique_id_broadcast():
    out = _run(_uid_fn)
    assert out[0] == out[1] == bytes(range(128))


def _shard_fn(rank, world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import bench_secondary
    from paper_2506_06190_b200.nat import row_range
    res = {}
    for n in (1, 7, 1280, 20480, 199692):
        res[n] = (row_range(n, rank, world), bench_secondary.shard(n, rank, world))
    res["mc"] = bench_secondary.mc_share(3, rank, world)
    res["geo"] = bench.geo_share(64, rank, world)
    return res


def test_row_listener_and_wavenumber_sharding_tile_exactly():
    out = _run(_shard_fn)
    for n in (1, 7, 1280, 20480, 199692):
        rows = [out[r][n][0] for r in range(WORLD)]
        assert rows == [out[r][n][1] for r in range(WORLD)]
        covered = np.concatenate([np.arange(a, b) for a, b in rows])
        assert np.array_equal(covered, np.arange(n))
        rpr = -(-n // WORLD)
        assert all(a == min(n, r * rpr) for r, (a, b) in enumerate(rows))
    ks = sorted(sum((out[r]["mc"] for r in range(WORLD)), []))
    assert ks == [0, 1, 2]
    # C4: every geometry on exactly one rank, equal counts (64 / world)
    geos = sorted(sum((out[r]["geo"] for r in range(WORLD)), []))
    assert geos == list(range(64)) and len({len(out[r]["geo"]) for r in range(WORLD)}) == 1


def _gmres_fn(rank, world):
    """Row-sharded GMRES with the library's protocol, arithmetic from the oracle."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import nat_inputs as I
    from oracle import bem, geometry, gmres
    from paper_2506_06190_b200.nat import row_range
    m = I.icosphere(2)
    geo = geometry.mesh_prepare(m.v, m.t)
    n = m.n_tri
    r0, r1 = row_range(n, rank, world)
    A_loc, b_loc = bem.assemble(m.v, m.t, geo, 2.0, I.neumann_rigid_z(m)[None], rows=np.arange(r0, r1))
    rpr = -(-n // world)

    def gather(v_loc):
        buf = torch.zeros(rpr, dtype=torch.complex128)
        buf[: v_loc.size] = torch.from_numpy(v_loc)
        parts = [torch.zeros(rpr, dtype=torch.complex128) for _ in range(world)]
        dist.all_gather(parts, buf)
        return torch.cat(parts).numpy()[:n]

    b = gather(b_loc[0])
    x, info = gmres.gmres(lambda z: gather(A_loc @ z), b, tol=1e-12, max_iter=200)
    return x, info["iters"]


def test_row_sharded_gmres_protocol_matches_single_process():
    import nat_inputs as I
    from oracle import bem, geometry, gmres
    out = _run(_gmres_fn)
    m = I.icosphere(2)
    geo = geometry.mesh_prepare(m.v, m.t)
    A, b = bem.assemble(m.v, m.t, geo, 2.0, I.neumann_rigid_z(m)[None])
    x, info = gmres.gmres(lambda z: A @ z, b[0], tol=1e-12, max_iter=200)
    for r in range(WORLD):
        assert out[r][1] == info["iters"]
        np.testing.assert_allclose(out[r][0], x, rtol=0, atol=1e-12 * np.abs(x).max())
    assert np.array_equal(out[0][0], out[1][0])   # replicated Arnoldi: identical on ranks


def _mc_gmres_fn(rank, world):
    """Row-sharded BEM-MC: every rank regenerates the same samples, forms its rows of the
    MC system (oracle arithmetic) and runs the replicated GMRES with an all-gather."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import nat_inputs as I
    from oracle import geometry, gmres, mc
    from paper_2506_06190_b200.nat import row_range
    m = I.icosphere(2)
    geo = geometry.mesh_prepare(m.v, m.t)
    M = 301
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, M, 5)
    g = I.neumann_constant(m)[tri]
    A, b = mc.system(y, n, g, 1.5, geo["total_area"])
    r0, r1 = row_range(M, rank, world)
    A_loc, b_loc = A[r0:r1], b[r0:r1]
    rpr = -(-M // world)

    def gather(v_loc):
        buf = torch.zeros(rpr, dtype=torch.complex128)
        buf[: v_loc.size] = torch.from_numpy(v_loc)
        parts = [torch.zeros(rpr, dtype=torch.complex128) for _ in range(world)]
        dist.all_gather(parts, buf)
        return torch.cat(parts).numpy()[:M]

    x, info = gmres.gmres(lambda z: gather(A_loc @ z), gather(b_loc), tol=1e-12, max_iter=200)
    return x, info["iters"], tri


def test_row_sharded_mc_protocol_matches_single_process():
    import nat_inputs as I
    from oracle import geometry, gmres, mc
    out = _run(_mc_gmres_fn)
    m = I.icosphere(2)
    geo = geometry.mesh_prepare(m.v, m.t)
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, 301, 5)
    A, b = mc.system(y, n, I.neumann_constant(m)[tri], 1.5, geo["total_area"])
    x, info = gmres.gmres(lambda z: A @ z, b, tol=1e-12, max_iter=200)
    for r in range(WORLD):
        assert np.array_equal(out[r][2], tri)          # identical samples on every rank
        assert out[r][1] == info["iters"]
        np.testing.assert_allclose(out[r][0], x, rtol=0, atol=1e-12 * np.abs(x).max())
    assert np.array_equal(out[0][0], out[1][0])


def _reduce_fn(rank, world):
    ms = torch.tensor([10.0 + rank], dtype=torch.float64)
    pairs = torch.tensor([1e9 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.all_reduce(pairs, op=dist.ReduceOp.SUM)
    return ms.item(), pairs.item()


def test_bench_reductions_max_time_sum_work():
    out = _run(_reduce_fn)
    for r in range(WORLD):
        assert out[r] == (11.0, 3e9)
