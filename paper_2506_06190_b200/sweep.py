"""The NAT training-data sweep (BASELINE.json configs[3], "C4") as a restartable job:
every scene geometry (8 heights x 8 sizes of a bowl over a passive slab)
through mesh preparation, the listener shell grid, BEM-MC with 64 wavenumbers
(8 materials x 8 modes, tol 1e-6 / 200 iterations) and the radiation of
the 64 fields to the listeners — the dataset step of P:166 — with one result file per
geometry and a manifest written last.

    python -m paper_2506_06190_b200.sweep --out DIR [--geometries 64] [--grid 64] [--workers 6]
    torchrun --nproc-per-node N -m paper_2506_06190_b200.sweep --out DIR     # geometries i mod N

Files in DIR:
  geo_XX.npy    fields, complex64 [64][P] (P = grid^3 listeners, wavenumber index 8 i_material + m)
  geo_XX.json   ks, GMRES iterations / convergence / true residual per system, listener grid
                frame, field file size — written AFTER the .npy (atomic rename): a geometry is
                done iff its .json exists and the .npy has the recorded size
  manifest.json the sweep's configuration and every geometry's record — written last (rank 0)
A rerun with the same DIR skips the geometries already done (resume).

This module only orchestrates: every step of the path runs in libnat's kernels (nat.py).
"""
from __future__ import annotations

import argparse
import json
import os
import queue
import threading
import time

import numpy as np

SEED = 20250606
M_SAMPLES = 2048


def geo_file(out_dir, gi, ext):
    return os.path.join(out_dir, f"geo_{gi:02d}.{ext}")


def is_done(out_dir, gi):
    """True iff geometry gi's record exists and its field file is complete."""
    js = geo_file(out_dir, gi, "json")
    if not os.path.exists(js):
        return False
    try:
        rec = json.load(open(js))
    except (OSError, ValueError):
        return False
    npy = geo_file(out_dir, gi, "npy")
    return os.path.exists(npy) and os.path.getsize(npy) == rec.get("field_bytes", -1)


def todo(out_dir, geo_ids):
    return [gi for gi in geo_ids if not is_done(out_dir, gi)]


def write_atomic(path, write):
    tmp = path + ".tmp"
    write(tmp)
    os.replace(tmp, path)


def save_geometry(out_dir, gi, field, rec):
    """field: complex numpy [n_k][P]; rec: JSON-serialisable dict.  .npy first, then .json."""
    f = np.ascontiguousarray(field.astype(np.complex64))

    def w_npy(tmp):
        with open(tmp, "wb") as fh:
            np.save(fh, f)
    write_atomic(geo_file(out_dir, gi, "npy"), w_npy)
    rec = dict(rec, field_bytes=os.path.getsize(geo_file(out_dir, gi, "npy")), field_dtype="complex64",
               field_shape=list(f.shape))
    write_atomic(geo_file(out_dir, gi, "json"), lambda tmp: json.dump(rec, open(tmp, "w"), indent=1))


def write_manifest(out_dir, n_geo, config):
    recs = {}
    for gi in range(n_geo):
        if not is_done(out_dir, gi):
            raise RuntimeError(f"geometry {gi} missing: the manifest is written only when all are done")
        recs[gi] = json.load(open(geo_file(out_dir, gi, "json")))
    man = {"config": config, "geometries": n_geo, "written": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "all_converged": all(all(r["converged"]) for r in recs.values()),
           "records": {str(k): v for k, v in recs.items()}}
    write_atomic(os.path.join(out_dir, "manifest.json"), lambda tmp: json.dump(man, open(tmp, "w"), indent=1))
    return man


def run_geometry(nat, torch, gi, grid, bufs):
    """One geometry through a1, a12, a8-a10, a11; returns (field on device, record)."""
    import nat_inputs as I
    m, g8, D = I.c4_geometry(gi)
    ks = [float(k) for k in I.c4_wavenumbers(D)]
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    g = torch.from_numpy(np.ascontiguousarray(np.tile(g8, (8, 1)))).cuda()
    geo = nat.nat_mesh_prepare(mesh)
    lis = nat.nat_listener_grid(geo.center, geo.bound_radius, grid, grid, grid)
    smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, ks, g, M_SAMPLES, seed=SEED, stream_id=gi,
                                                      prec="fp32", tol=1e-6, plan=bufs["mc"])
    gs = nat.nat_mc_gather_neumann(g, stri)
    src = nat.nat_mc_sources(smp, geo.total_area, p, gs, center=geo.center)
    out = nat.nat_radiate_field(src, ks, lis, "fp32", plan=bufs["rad"])
    rec = {"geometry": gi, "n_tri": m.n_tri, "bowl_diameter_m": D, "ks": ks, "M": M_SAMPLES, "seed": SEED,
           "stream_id": gi, "grid": [grid] * 3, "center": list(geo.center), "bound_radius": geo.bound_radius,
           "listener_shell": [1.5, 3.0],
           "iters": [i["iters"] for i in infos], "converged": [bool(i["converged"]) for i in infos],
           "rel_residual": [i["rel_residual"] for i in infos]}
    return out, rec


def run(out_dir, n_geo=64, grid=64, workers=6, rank=0, world=1, log=print):
    import torch
    from paper_2506_06190_b200 import nat
    nat.sweep_tuning()
    nat.lib()
    os.makedirs(out_dir, exist_ok=True)
    mine = [gi for gi in range(n_geo) if gi % world == rank]
    pending = todo(out_dir, mine)
    log(f"[sweep] rank {rank}/{world}: {len(mine)} geometries, {len(mine) - len(pending)} already done")
    q = queue.Queue()
    for gi in pending:
        q.put(gi)
    err = []

    def worker():
        try:
            s = torch.cuda.Stream()
            bufs = {"mc": nat.McPlan(M_SAMPLES, 64, "fp32", 200, "cuda"),
                    "rad": nat.RadiatePlan(M_SAMPLES, 64, grid ** 3, "fp32", "cuda")}
            with torch.cuda.stream(s):
                while True:
                    try:
                        gi = q.get_nowait()
                    except queue.Empty:
                        return
                    t0 = time.perf_counter()
                    out, rec = run_geometry(nat, torch, gi, grid, bufs)
                    field = out.cpu().numpy()          # synchronises this stream
                    rec["seconds"] = time.perf_counter() - t0
                    save_geometry(out_dir, gi, field, rec)
                    log(f"[sweep] geometry {gi}: {rec['seconds']:.2f} s, iterations "
                        f"{min(rec['iters'])}..{max(rec['iters'])}, converged {sum(rec['converged'])}/64")
        except BaseException as ex:  # pragma: no cover - re-raised below
            err.append(ex)

    ths = [threading.Thread(target=worker) for _ in range(max(1, workers))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]
    return mine


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--geometries", type=int, default=64)
    ap.add_argument("--grid", type=int, default=64)
    ap.add_argument("--workers", type=int, default=6)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    import torch
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
    run(a.out, a.geometries, a.grid, a.workers, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    if rank == 0:
        man = write_manifest(a.out, a.geometries, {"config": "C4", "geometries": a.geometries, "grid": a.grid,
                                                   "M": M_SAMPLES, "seed": SEED, "world": world})
        print(f"[sweep] manifest written: {a.geometries} geometries, all converged: {man['all_converged']}")
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
