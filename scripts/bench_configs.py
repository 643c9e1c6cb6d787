"""Per-config measurements beside bench.py's C2 step (BASELINE.json configs C1, C3, C4, C5
and the NEXT-3 Poisson sampler): device time with CUDA events (1 warm-up + 3 timed runs,
median), rates in the units of SURVEY.md §8(d).  Writes one JSON object to stdout.

    python scripts/bench_configs.py > profiles/r01_configs.json
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import nat_inputs as I  # noqa: E402
from paper_2506_06190_b200 import nat  # noqa: E402

R_PIPE = 148 * 128 * 1965e6 / 24.0


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts), out


def c1(prec):
    m = I.icosphere(3)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    g = torch.ones(1, m.n_tri, dtype=torch.complex128, device="cuda")
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 4, 4, 4)

    def run():
        geo = nat.nat_mesh_prepare(mesh)
        near = nat.nat_bem_near_list(mesh, geo)
        A, b = nat.nat_bem_assemble(mesh, geo, near, 1.0, g, prec=prec)
        x, info = nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6 if prec == "fp32" else 1e-12)
        src = nat.nat_bem_sources(mesh, geo, x[None], g)
        return nat.nat_radiate_field(src, [1.0], lis, prec)

    t, out = timed(run)
    x = lis.T.cpu().numpy()
    r = np.linalg.norm(x, axis=1)
    exact = np.exp(1j * (r - 1.0)) / ((1j - 1.0) * r)          # pulsating sphere, a = g = k = 1
    err = np.linalg.norm(out[0].cpu().numpy() - exact) / np.linalg.norm(exact)
    return {"seconds": t, "analytic_rel_l2": float(err), "note": "mesh prep + near list + assembly + GMRES + "
            "radiation to 4^3 listeners, icosphere L3 (1280 tri), g = 1, k = 1"}


def c3():
    m = I.bowl()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    ks = list(I.c3_wavenumbers())
    g = torch.from_numpy(I.neumann_harmonics(m, 32)).cuda()
    M = 4096
    plan = nat.McPlan(M, 32, "fp32", 200, "cuda")
    t, (smp, stri, p, infos) = timed(lambda: nat.nat_mc_surface_pressure(mesh, geo, ks, g, M, seed=I.SEED,
                                                                         prec="fp32", plan=plan))
    iters = [i["iters"] for i in infos]
    pairs = sum(M * (M - 1) * (1 + it) for it in iters)
    gs = nat.nat_mc_gather_neumann(g, stri)
    src = nat.nat_mc_sources(smp, geo.total_area, p, gs, center=geo.center)
    lis = nat.nat_listener_grid(geo.center, geo.bound_radius, 32, 32, 32)
    rplan = nat.RadiatePlan(M, 32, lis.shape[1], "fp32", "cuda")
    out = torch.empty(32, lis.shape[1], dtype=torch.complex128, device="cuda")
    tr, _ = timed(lambda: nat.nat_radiate_field(src, ks, lis, "fp32", out=out, plan=rplan))
    tp, (psmp, pstri, r) = timed(lambda: nat.nat_mc_poisson_sample(mesh, geo, M, seed=I.SEED))
    Mp = psmp.shape[1]
    plan_p = nat.McPlan(Mp, 32, "fp32", 200, "cuda")
    tq, (_, _, _, pinfos) = timed(lambda: nat.nat_mc_surface_pressure(
        mesh, geo, ks, g, Mp, prec="fp32", samples_in=psmp.contiguous(), sample_tri_in=pstri, plan=plan_p))
    return {"mc_solve_seconds": t, "mc_iters": iters, "mc_pair_evals_per_s": pairs / t,
            "mc_frac_R_pipe": pairs / t / R_PIPE,
            "radiation_seconds": tr, "radiation_pair_modes_per_s": M * lis.shape[1] * 32 / tr,
            "radiation_listener_pt_modes_per_s": lis.shape[1] * 32 / tr,
            "poisson_sample_seconds": tp, "poisson_M": Mp, "poisson_r": r,
            "mc_solve_poisson_seconds": tq, "mc_iters_poisson": [i["iters"] for i in pinfos],
            "note": "bowl 49,664 tri, 32 modes (k a = 0.5 .. 8), M = 4096 uniform samples, tol 1e-6; radiation "
                    "of the 32 modes fused to the 32^3 grid; Poisson-disk sampler (M_target 4096) and the MC "
                    "solve on its samples"}


def c4(gi=0):
    m, g8, D = I.c4_geometry(gi)
    ks = list(I.c4_wavenumbers(D))
    g = torch.from_numpy(np.tile(g8, (8, 1))).cuda()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    M = 2048
    plan = nat.McPlan(M, 64, "fp32", 200, "cuda")
    t, (smp, stri, p, infos) = timed(lambda: nat.nat_mc_surface_pressure(mesh, geo, ks, g, M, seed=I.SEED,
                                                                         stream_id=gi, prec="fp32", plan=plan))
    iters = [i["iters"] for i in infos]
    gs = nat.nat_mc_gather_neumann(g, stri)
    src = nat.nat_mc_sources(smp, geo.total_area, p, gs, center=geo.center)
    lis = nat.nat_listener_grid(geo.center, geo.bound_radius, 64, 64, 64)
    rplan = nat.RadiatePlan(M, 64, lis.shape[1], "fp32", "cuda")
    out = torch.empty(64, lis.shape[1], dtype=torch.complex128, device="cuda")
    tr, _ = timed(lambda: nat.nat_radiate_field(src, ks, lis, "fp32", out=out, plan=rplan))
    pm = M * lis.shape[1] * 64
    return {"n_tri": m.n_tri, "mc_solve_seconds": t, "mc_iters_min_max": [min(iters), max(iters)],
            "radiation_seconds": tr, "radiation_pair_modes_per_s": pm / tr,
            "radiation_listener_pt_modes_per_s": lis.shape[1] * 64 / tr,
            "radiation_frac_R_sfu_multimode": pm / tr / 2.31e12,
            "note": f"geometry {gi} (bowl over slab), M = 2048, 64 wavenumbers batched; radiation of all 64 fused "
                    "to the 64^3 grid (roofline per pair-mode for fused modes: R_sfu 2.31e12, SURVEY §8d)"}


def c4_sweep(n_geo=64):
    """C4 end to end on one GPU: all 64 scene geometries (8 heights x 8 sizes), each with
    64 wavenumbers (8 materials x 8 modes): mesh preparation, Philox samples, the batched
    MC solve and the fused radiation to its 64^3 listener grid.  Meshes are uploaded before
    the timed region; device time with CUDA events over the whole sweep."""
    scenes = []
    for gi in range(n_geo):
        m, g8, D = I.c4_geometry(gi)
        scenes.append((gi, nat.Mesh.from_numpy(m.v, m.t), torch.from_numpy(np.tile(g8, (8, 1))).cuda(),
                       list(I.c4_wavenumbers(D)), m.n_tri))
    M = 2048
    plan = nat.McPlan(M, 64, "fp32", 200, "cuda")
    P = 64 ** 3
    rplan = nat.RadiatePlan(M, 64, P, "fp32", "cuda")
    out = torch.empty(64, P, dtype=torch.complex128, device="cuda")
    iters = []

    def run():
        for gi, mesh, g, ks, _ in scenes:
            geo = nat.nat_mesh_prepare(mesh)
            smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, ks, g, M, seed=I.SEED, stream_id=gi,
                                                              prec="fp32", plan=plan)
            iters.append(sum(i["iters"] for i in infos))
            src = nat.nat_mc_sources(smp, geo.total_area, p, nat.nat_mc_gather_neumann(g, stri), center=geo.center)
            lis = nat.nat_listener_grid(geo.center, geo.bound_radius, 64, 64, 64)
            nat.nat_radiate_field(src, ks, lis, "fp32", out=out, plan=rplan)
        return None

    t, _ = timed(run, reps=1)
    n = len(scenes)
    return {"geometries": n, "wavenumbers_per_geometry": 64, "configs": n * 8, "seconds": t,
            "seconds_per_geometry": t / n, "listener_pt_modes_per_s": n * 64 * P / t,
            "mean_gmres_iters_per_system": float(np.mean(iters[-n:]) / 64),
            "note": "the NAT training-data sweep (BASELINE configs[3]) on one GPU: 64 geometries x 64 "
                    "wavenumbers = 512 configs x 8 modes; per geometry mesh prep + M = 2048 samples + batched MC "
                    "solve + fused radiation to 64^3 listeners (262,144 x 64 field values); 8 GPUs deal geometries"}


def c5(rows=1024):
    m = I.cubed_sphere(129)
    gt = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    near = nat.nat_bem_near_list(mesh, geo, 0, rows)
    A = torch.empty(rows, m.n_tri, dtype=torch.complex128, device="cuda")
    ta, _ = timed(lambda: nat.nat_bem_assemble(mesh, geo, near, 8.0, gt, prec="fp64", A=A, lda=m.n_tri))
    nS = int((near.cls == 1).sum().item())
    pairs = rows * m.n_tri * 3 + nS * 448 + (near.nnz - nS) * 28 + rows * 48
    x = torch.from_numpy(I.random_complex(m.n_tri, 1)).cuda()
    y = torch.empty(rows, dtype=torch.complex128, device="cuda")
    tg, _ = timed(lambda: nat.nat_bem_matvec(A, x, n=m.n_tri, out=y), reps=5)
    pv = torch.from_numpy(I.random_complex(m.n_tri, 2)[None]).cuda()
    src = nat.nat_bem_sources(mesh, geo, pv, gt)
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 8, 8, 8)
    tr, _ = timed(lambda: nat.nat_radiate_field(src, [8.0], lis, "fp64"), reps=1)
    return {"rows": rows, "n_tri": m.n_tri, "fp64_assembly_seconds": ta, "fp64_assembly_pair_evals_per_s": pairs / ta,
            "c128_gemv_seconds": tg, "c128_gemv_GBps": rows * m.n_tri * 16 / tg / 1e9,
            "fp64_radiation_seconds": tr, "fp64_radiation_listener_pts_per_s": lis.shape[1] / tr,
            "fp64_radiation_pair_evals_per_s": 3 * m.n_tri * lis.shape[1] / tr,
            "note": "cubed sphere 199,692 tri, one rank's row block at ka = 8 (fp64, c128 matrix), its GEMV, fp64 "
                    "radiation of all 599,076 sources to an 8^3 grid"}


def _mf_case(m, ka, prec, g):
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    near = nat.nat_bem_near_list(mesh, geo)
    gt = torch.from_numpy(g[None]).cuda()
    tp, (op, rhs) = timed(lambda: nat.nat_bem_mf_prepare(mesh, geo, near, ka, gt, prec=prec), reps=1)
    return mesh, geo, near, gt, op, rhs, tp


def c5_mf(ka=8.0):
    """NEXT-3: C5 (199,692 tri, fp64, tol 1e-12) solved on ONE GPU with the matrix-free
    operator (the stored matrix would be 638 GB)."""
    m = I.cubed_sphere(129)
    g = I.neumann_rigid_z(m)
    mesh, geo, near, gt, op, rhs, tp = _mf_case(m, ka, "fp64", g)
    ts, (x, info) = timed(lambda: nat.nat_bem_mf_solve(op, rhs[0], tol=1e-12), reps=1)
    x0 = torch.from_numpy(I.random_complex(m.n_tri, 1)).cuda()
    tm, _ = timed(lambda: nat.nat_bem_mf_matvec(op, x0), reps=2)
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 8, 8, 4)
    src = nat.nat_bem_sources(mesh, geo, x[None], gt)
    p = nat.nat_radiate_field(src, [ka], lis, "fp64")[0].cpu().numpy()
    from oracle import analytic
    pe = analytic.oscillating_sphere(lis.T.cpu().numpy(), ka)
    far = 3.0 * m.n_tri * m.n_tri
    return {"n_tri": m.n_tri, "ka": ka, "prepare_seconds": tp, "solve_seconds_per_mode": ts,
            "iters": info["iters"], "rel_residual": info["rel_residual"],
            "matvec_seconds": tm, "far_pair_evals_per_matvec": far, "fp64_far_pair_evals_per_s": far / tm,
            "solve_matvec_device_seconds": info["t_matvec_s"],
            "analytic_rel_l2": float(np.linalg.norm(p - pe) / np.linalg.norm(pe)),
            "note": "cubed sphere 199,692 tri, dipole, ka = 8, fp64 matrix-free operator on one GPU: near/self "
                    "corrections prepared once (c128 [nnz]), far rule re-evaluated in every product; GMRES tol "
                    "1e-12; field at an 8x8x4 shell grid vs the analytic oscillating sphere"}


def c2_mf(ka=8.0):
    """NEXT-3 at the C2 size (fp32): matrix-free product vs the stored-matrix GEMV."""
    m = I.icosphere(5)
    g = I.neumann_rigid_z(m)
    mesh, geo, near, gt, op, rhs, tp = _mf_case(m, ka, "fp32", g)
    x0 = torch.from_numpy(I.random_complex(m.n_tri, 1)).cuda()
    tm, _ = timed(lambda: nat.nat_bem_mf_matvec(op, x0), reps=5)
    ts, (x, info) = timed(lambda: nat.nat_bem_mf_solve(op, rhs[0], tol=1e-6), reps=3)
    far = 3.0 * m.n_tri * m.n_tri
    return {"n_tri": m.n_tri, "ka": ka, "prepare_seconds": tp, "matvec_seconds": tm,
            "far_pair_evals_per_s": far / tm, "far_frac_R_pipe": far / tm / R_PIPE,
            "solve_seconds": ts, "iters": info["iters"],
            "note": "icosphere L5, dipole, fp32 matrix-free product (far rule re-evaluated: 1.26e9 pair-evals) "
                    "against the stored c64 GEMV of r01 (3.36 GB at HBM speed, ~0.49 ms)"}


def gal_c2(ka=8.0):
    """NEXT-2 at the C2 size: fp32 Galerkin assembly + GMRES of the dipole, analytic error."""
    m = I.icosphere(5)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    o = nat.quad_opts(galerkin=True)
    near = nat.nat_bem_near_list(mesh, geo, opts=o)
    g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
    A = torch.empty(m.n_tri, m.n_tri, dtype=torch.complex64, device="cuda")
    ta, (A, b) = timed(lambda: nat.nat_bem_assemble(mesh, geo, near, ka, g, prec="fp32", A=A, opts=o))
    ts, (x, info) = timed(lambda: nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6))
    cls = near.cls.cpu().numpy()
    tri = m.t
    rp = near.row_ptr.cpu().numpy()
    col = near.col.cpu().numpy()
    rows = np.repeat(np.arange(m.n_tri), np.diff(rp))
    shared = (tri[rows][:, :, None] == tri[col][:, None, :]).any(axis=2).sum(axis=1)
    n_edge, n_vert = int((shared == 2).sum()), int((shared == 1).sum())
    n_far = m.n_tri * (m.n_tri - 1) - near.nnz
    pairs = n_far * 9 + int((cls == 2).sum()) * 784 + n_edge * 5 * 256 + n_vert * 2 * 256 + m.n_tri * 6 * 256
    lis = nat.nat_listener_grid((0, 0, 0), 1.0, 8, 8, 2)
    p = nat.nat_radiate_field(nat.nat_bem_sources(mesh, geo, x[None], g), [ka], lis)[0].cpu().numpy()
    from oracle import analytic
    pe = analytic.oscillating_sphere(lis.T.cpu().numpy(), ka)
    return {"assembly_seconds": ta, "assembly_pair_evals": pairs, "assembly_pair_evals_per_s": pairs / ta,
            "assembly_frac_R_pipe": pairs / ta / R_PIPE, "solve_seconds": ts, "iters": info["iters"],
            "analytic_rel_l2": float(np.linalg.norm(p - pe) / np.linalg.norm(pe)),
            "note": "icosphere L5 (20,480 tri), dipole, ka = 8, fp32 Galerkin P0: far 3x3 tensor points, class N "
                    "28x28, Sauter-Schwab order 4 (identical 1536 / edge 1280 / vertex 512 points)"}


def bm_c2():
    """NEXT-1 at the C2 size: fp32 Burton-Miller assembly + GMRES of the dipole at ka = 8."""
    m = I.icosphere(5)
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    geo = nat.nat_mesh_prepare(mesh)
    near = nat.nat_bem_near_list(mesh, geo)
    g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
    A = torch.empty(m.n_tri, m.n_tri, dtype=torch.complex64, device="cuda")
    o = nat.quad_opts(burton_miller=True)
    ta, (A, b) = timed(lambda: nat.nat_bem_assemble(mesh, geo, near, 8.0, g, prec="fp32", A=A, opts=o))
    ts, (x, info) = timed(lambda: nat.nat_bem_solve(A, b[0], m.n_tri, tol=1e-6))
    nS = int((near.cls == 1).sum().item())
    pairs = m.n_tri * m.n_tri * 3 + nS * 448 + (near.nnz - nS) * 28
    return {"assembly_seconds": ta, "assembly_bm_pair_evals_per_s": pairs / ta, "solve_seconds": ts,
            "iters": info["iters"], "note": "icosphere L5 (20,480 tri), dipole, ka = 8, fp32, Burton-Miller "
            "(each pair evaluates G, dG/dn_y, dG/dn_x and d2G/dn_x dn_y)"}


def main():
    torch.cuda.set_device(0)
    nat.lib()
    res = {"device": torch.cuda.get_device_name(0)}
    sel = set(sys.argv[1:])
    for name, fn in (("C1_fp32", lambda: c1("fp32")), ("C1_fp64", lambda: c1("fp64")), ("C3", c3), ("C4", c4),
                     ("C5", c5), ("BM_C2", bm_c2), ("C5_MF", c5_mf), ("C2_MF", c2_mf), ("GAL_C2", gal_c2),
                     ("C4_SWEEP", c4_sweep)):
        if sel and name not in sel:
            continue
        try:
            res[name] = fn()
        except Exception as ex:  # pragma: no cover - reported, not fatal
            res[name] = {"error": repr(ex)}
        print(f"[configs] {name} done", file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
