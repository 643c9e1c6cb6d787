#!/usr/bin/env python3
"""bench.py — the NAT Helmholtz boundary-integral hot path on B200 (sm_100a).

One *step* = the NAT training-data sweep, BASELINE.json configs[3] ("C4"), the
largest configuration of the path that runs on one GPU and the one the north star's
throughput is quoted on ("synthetic meshes and modal/Neumann data shaped like the
paper's scenes (object position, size and material sweeps, with listener grids)"):

  64 scene geometries = 8 heights x 8 sizes of a bowl over a passive slab
  (19,584 triangles each), per geometry 64 wavenumbers
  (8 materials x 8 modes: 512 configs x 8 modes), and per geometry
    a1  mesh preparation,
    a12 the 64^3 listener shell grid (r = 1.5 .. 3 R),
    a8  M = 2048 Philox samples (P:385's "2K"), a9 the MC right-hand sides,
    a10 the batched GMRES over the matrix-free MC operator (64 systems, tol 1e-6),
    a11 radiation of the 64 solutions to the 262,144 listeners (fused wavenumbers).

Geometries are dealt to ranks as i mod N with no collective ("scaling": "strong": the
total work is fixed).  Inside a rank, W worker threads (each with its own CUDA stream and
workspaces) take geometries from a queue, so one geometry's HBM-bound Krylov kernels
overlap another's MUFU/FP32-bound pair kernels.

value = pair-evaluations x wavenumbers of the step (MC right-hand sides 64 M (M-1), MC
operator sum_systems iterations x M (M-1), radiation 64 M P per geometry) / device time,
in Gpair-evals/s; listener_pts_per_s = listener points x wavenumbers per second.
e2e = the same with every geometry's mesh and Neumann data copied from pinned host memory
and every radiated field (64 x 262,144 c128 = 268 MB) copied back to pinned host memory
inside the timed region.  Secondary lines (C2 dense BEM + BEM-MC, C3 modal MC) are in
"secondary" (bench_secondary.py).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nat|reference]
"""
import argparse
import json
import math
import concurrent.futures
import gc
import os
import queue
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Helmholtz kernel Gpair-evals/s and listener pts/s vs FP32 roofline at 1/2/4/8 B200"
UNIT = "Gpair-evals/s"
N_GEO, N_K, M_C4 = 64, 64, 2048
GRID = (64, 64, 64)
P_LIS = GRID[0] * GRID[1] * GRID[2]
SM_COUNT, MAX_MHZ = 148, 1965.0
WORKLOAD = ("C4: NAT training-data sweep, 64 geometries (bowl over slab, 19,584 tri; 8 heights x 8 sizes) x "
            "64 wavenumbers (8 materials x 8 modes = 512 configs x 8 modes); per geometry mesh prep, 64^3 "
            "listener shell grid, BEM-MC with M = 2048 Philox samples (64 systems batched, GMRES tol 1e-6), "
            "radiation of the 64 fields to the 262,144 listeners")

# Per pair-evaluation instruction counts of the minimal formulation (SURVEY.md §8(d),
# Appendix B.5): FP32-pipe instructions shared by the n wavenumbers of a launch (d, r^2,
# d.n, rho^2, q, r) + per wavenumber (kr, range reduction, coefficients, accumulation);
# MUFU: rsqrt shared, sin + cos per wavenumber.  kind 0 = G + dG (radiation), 1 = dG only
# (MC operator), 2 = G only (MC right-hand side).
FP32_SHARED = {0: 12.0, 1: 12.0, 2: 7.0}
FP32_PER_K = {0: 12.0, 1: 10.0, 2: 8.0}


def sm_clk_per_pair(kind, n):
    """Binding SM-clocks per pair-evaluation x wavenumber for a launch of n wavenumbers:
    max(FP32 instr / 128 lanes, MUFU / 16 units) (the MUFU binds for every kind)."""
    fp32 = FP32_SHARED[kind] / n + FP32_PER_K[kind]
    mufu = 1.0 / n + 2.0
    return max(fp32 / 128.0, mufu / 16.0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nat", choices=["nat", "reference"])
    ap.add_argument("--workers", type=int, default=int(os.environ.get("NAT_BENCH_WORKERS", "0")),
                    help="worker threads per GPU (0: 6, or every geometry of the rank at once when it has <= 8)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile-count", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--geometries", type=int, default=N_GEO, help="sweep subset (tuning only)")
    return ap.parse_args()


def geo_share(n_geo, rank, world):
    """C4 geometries of one rank: i mod world == rank (no collective)."""
    return [gi for gi in range(n_geo) if gi % world == rank]


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# ----------------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ----------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append(mhz)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception as ex:
                self.err = str(ex)
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------------
# the C4 sweep (the step)
# ----------------------------------------------------------------------------------
def load_c4_host(geo_ids):
    import nat_inputs as I
    out = {}
    for gi in geo_ids:
        m, g8, D = I.c4_geometry(gi)
        out[gi] = dict(v=np.ascontiguousarray(m.v.T), t=np.ascontiguousarray(m.t.T.astype(np.int32)),
                       g=np.ascontiguousarray(np.tile(g8, (8, 1))), ks=[float(k) for k in I.c4_wavenumbers(D)],
                       n_tri=m.n_tri, n_vert=m.v.shape[0])
    return out


class Worker:
    """One host thread's CUDA streams, workspaces and output buffers.  The MC solve runs on a
    high-priority stream and the radiation on a low-priority one: the solve is a chain of
    ~120-170 dependent small launches whose latency sets the geometry's time, the radiation
    is a bulk MUFU-bound pass that can fill whatever the solves leave idle, and geometry
    q + 1's solve overlaps geometry q's radiation (per-geometry buffers double-buffered)."""

    def __init__(self, nat, torch, n_vert, n_tri, e2e_out):
        dev = torch.device("cuda")
        prio = os.environ.get("NAT_BENCH_PRIO", "1") != "0"   # A/B: equal priorities
        self.stream = torch.cuda.Stream(priority=-5 if prio else 0)   # clamped to the device's highest priority
        self.rad_stream = torch.cuda.Stream(priority=0)
        self.copy_stream = torch.cuda.Stream()
        self.mc_plan = nat.McPlan(M_C4, N_K, "fp32", 200, dev)
        self.rad_plan = nat.RadiatePlan(M_C4, N_K, P_LIS, "fp32", dev)
        # per-geometry buffers read by the radiation: two slots
        self.smp = [torch.empty(6, M_C4, dtype=torch.float64, device=dev) for _ in range(2)]
        self.stri = [torch.empty(M_C4, dtype=torch.int32, device=dev) for _ in range(2)]
        self.p = [torch.empty(N_K, M_C4, dtype=torch.complex128, device=dev) for _ in range(2)]
        self.gs = [torch.empty(N_K, M_C4, dtype=torch.complex128, device=dev) for _ in range(2)]
        self.lis = [torch.empty(3, P_LIS, dtype=torch.float64, device=dev) for _ in range(2)]
        self.solved = [torch.cuda.Event() for _ in range(2)]
        self.radiated = [torch.cuda.Event() for _ in range(2)]
        self.gslot = 0
        # double-buffered field: the D2H of geometry q overlaps the radiation of q + 1
        self.out = [torch.empty(N_K, P_LIS, dtype=torch.complex128, device=dev) for _ in range(2)]
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.slot = 0
        # staging mesh / Neumann buffers of the e2e pass (inputs copied from pinned host)
        self.mesh = nat.Mesh(torch.empty(3, n_vert, dtype=torch.float64, device=dev),
                             torch.empty(3, n_tri, dtype=torch.int32, device=dev))
        self.g = torch.empty(N_K, n_tri, dtype=torch.complex128, device=dev)
        self.host_out = torch.empty(N_K, P_LIS, dtype=torch.complex128).pin_memory() if e2e_out else None


class Sweep:
    def __init__(self, nat, torch, rank, world, n_workers, n_geo=N_GEO, e2e=True):
        self.nat, self.torch = nat, torch
        self.geo_ids = geo_share(n_geo, rank, world)
        self.host = load_c4_host(self.geo_ids)
        h0 = self.host[self.geo_ids[0]]
        self.n_tri, self.n_vert = h0["n_tri"], h0["n_vert"]
        dev = torch.device("cuda")
        # device-resident inputs (the `value` pass) and pinned host copies (the e2e pass)
        self.dmesh, self.dg, self.pinned = {}, {}, {}
        for gi, h in self.host.items():
            self.dmesh[gi] = nat.Mesh(torch.from_numpy(h["v"]).to(dev), torch.from_numpy(h["t"]).to(dev))
            self.dg[gi] = torch.from_numpy(h["g"]).to(dev)
            if e2e:
                self.pinned[gi] = tuple(torch.from_numpy(h[k]).pin_memory() for k in ("v", "t", "g"))
        self.workers = [Worker(nat, torch, self.n_vert, self.n_tri, e2e) for _ in range(n_workers)]
        self.verbose = bool(os.environ.get("NAT_BENCH_VERBOSE"))
        self.cost = {}   # host seconds per geometry in the last pass (NAT_BENCH_VERBOSE)
        self.pool, self.pool_size = None, 0
        self.lock = threading.Lock()

    def _geometry(self, w, gi, host_io, rec, keep=None, serial=False):
        nat, torch = self.nat, self.torch
        h = self.host[gi]
        if host_io:   # inputs from pinned host memory (e2e)
            pv, pt, pg = self.pinned[gi]
            w.mesh.vxyz.copy_(pv, non_blocking=True)
            w.mesh.tri.copy_(pt, non_blocking=True)
            w.g.copy_(pg, non_blocking=True)
            mesh, g = w.mesh, w.g
        else:
            mesh, g = self.dmesh[gi], self.dg[gi]
        k = w.gslot
        w.stream.wait_event(w.radiated[k])   # slot k's previous radiation has read its buffers
        geo = nat.nat_mesh_prepare(mesh)                                                       # a1
        nat.nat_listener_grid(geo.center, geo.bound_radius, *GRID, out=w.lis[k])               # a12
        smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, h["ks"], g, M_C4, seed=20250606, stream_id=gi,
                                                          prec="fp32", tol=1e-6, plan=w.mc_plan,
                                                          out=(w.smp[k], w.stri[k], w.p[k]))   # a8-a10
        nat.nat_mc_gather_neumann(g, stri, out=w.gs[k])
        src = nat.nat_mc_sources(smp, geo.total_area, p, w.gs[k], center=geo.center)
        w.solved[k].record(w.stream)
        out = w.out[w.slot]
        rs = w.stream if serial else w.rad_stream   # serial: the kernel-timer pass (no overlap)
        if rs is not w.stream:   # the source arrays were allocated on w.stream: keep them alive for rs
            for t in (src.xyz, src.nrm, src.w, src.p, src.g):
                t.record_stream(rs)
        with torch.cuda.stream(rs):
            rs.wait_event(w.solved[k])
            if host_io:
                rs.wait_event(w.copied[w.slot])   # the slot's previous D2H is done
            nat.nat_radiate_field(src, h["ks"], w.lis[k], "fp32", out=out, plan=w.rad_plan)   # a11
            if keep is not None:   # tests: a copy of the field, taken in stream order
                keep[gi] = out.clone()
            w.radiated[k].record(rs)
        w.gslot ^= 1
        if host_io:   # field -> pinned host on the copy stream
            w.copy_stream.wait_event(w.radiated[k])
            with torch.cuda.stream(w.copy_stream):
                w.host_out.copy_(out, non_blocking=True)
                w.copied[w.slot].record()
            w.slot ^= 1
        iters = [i["iters"] for i in infos]
        conv = all(i["converged"] for i in infos)
        mm = M_C4 * (M_C4 - 1)
        with self.lock:
            rec["mc_rhs"] += N_K * mm
            rec["mc_op"] += sum(iters) * mm
            rec["rad"] += N_K * M_C4 * P_LIS
            rec["lis_pt_modes"] += N_K * P_LIS
            rec["iters"].extend(iters)
            rec["converged"] = rec["converged"] and conv
            rec["unconverged"] += sum(1 for i in infos if not i["converged"])
            rec["max_rel_residual"] = max(rec["max_rel_residual"], max(i["rel_residual"] for i in infos))
            rec["geometries"] += 1
            rec["h2d"] += (h["v"].nbytes + h["t"].nbytes + h["g"].nbytes) if host_io else 0
            rec["d2h"] += out.numel() * 16 if host_io else 0

    def run(self, host_io=False, n_workers=None, geo_ids=None, keep=None, serial=False):
        """One step: every geometry of this rank through a1-a12, W worker threads."""
        torch = self.torch
        ids = self.geo_ids if geo_ids is None else geo_ids
        ws = self.workers[: (n_workers or len(self.workers))]
        rec = dict(mc_rhs=0, mc_op=0, rad=0, lis_pt_modes=0, iters=[], converged=True, geometries=0, h2d=0, d2h=0,
                   unconverged=0, max_rel_residual=0.0)
        q = queue.Queue()
        for gi in ids:
            q.put(gi)
        cur = torch.cuda.current_stream()
        ready = torch.cuda.Event()
        ready.record(cur)
        err = []

        t_run = time.perf_counter()
        spans = {}

        def loop(w):
            t_start = time.perf_counter() - t_run
            n_done = 0
            try:
                with torch.cuda.stream(w.stream):
                    w.stream.wait_event(ready)
                    w.rad_stream.wait_event(ready)
                    while True:
                        try:
                            gi = q.get_nowait()
                        except queue.Empty:
                            return
                        t0 = time.perf_counter()
                        self._geometry(w, gi, host_io, rec, keep, serial)
                        dt = time.perf_counter() - t0
                        n_done += 1
                        with self.lock:
                            self.cost[gi] = dt
                            if self.verbose:
                                rec.setdefault("host_s", []).append((round(dt, 3), gi))
                                spans[id(w)] = (round(t_start, 3), round(time.perf_counter() - t_run, 3), n_done)
            except BaseException as ex:   # re-raised on the main thread
                err.append(ex)

        if len(ws) == 1:
            loop(ws[0])
        else:
            # persistent threads: libnat keeps per-thread pinned rings and events (created on a
            # thread's first solve, released when it exits), so threads must outlive the steps
            if self.pool is None or self.pool_size < len(ws):
                self.pool = concurrent.futures.ThreadPoolExecutor(max_workers=len(ws))
                self.pool_size = len(ws)
            for f in [self.pool.submit(loop, w) for w in ws]:
                f.result()
        if err:
            raise err[0]
        if self.verbose:
            print(f"[bench] worker spans (start, end, geometries): {sorted(spans.values())}", file=sys.stderr)
        for w in ws:
            cur.wait_stream(w.stream)
            cur.wait_stream(w.rad_stream)
            cur.wait_stream(w.copy_stream)
        return rec


def step_pairs(rec):
    return rec["mc_rhs"] + rec["mc_op"] + rec["rad"]


def merge(a, b):
    if a is None:
        return dict(b, iters=list(b["iters"]))
    out = {}
    for k, v in b.items():
        out[k] = (a[k] and v) if k == "converged" else max(a[k], v) if k == "max_rel_residual" else a[k] + v
    return out


# ----------------------------------------------------------------------------------
# oracle timing (cpu_baseline and --impl reference): a bounded sample of the C4 step
# ----------------------------------------------------------------------------------
def _oracle_job(args):
    """One worker process's share of the sample: the oracle as it stands on geometry
    gi's a1 + a8, then `rows` rows of the MC operator and right-hand side for every one
    of the 64 wavenumbers and the radiation of the 64 modes to `n_lis` listeners."""
    gi, rows, n_lis = args
    import nat_inputs as I
    from oracle import geometry, kernel, listeners, mc, radiate
    m, g8, D = I.c4_geometry(gi)
    ks = I.c4_wavenumbers(D)
    t0 = time.perf_counter()
    geo = geometry.mesh_prepare(m.v, m.t)
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, M_C4, 20250606, gi)
    eps = mc.default_eps(geo["total_area"], M_C4)
    w = mc.weight(geo["total_area"], M_C4, eps)
    p = np.ones(M_C4, dtype=complex)
    pairs = 0
    for i in rows:
        j = np.arange(M_C4) != i
        for q, k in enumerate(ks):
            g = g8[q % 8][tri]
            _ = 0.5 * p[i] - w * np.sum(kernel.green_dn_y(y[i], y[j], n[j], k) * p[j])
            _ = -w * np.sum(kernel.green(y[i], y[j], k) * g[j]) - 0.5 * eps * g[i]
            pairs += 2 * (M_C4 - 1)
    L = listeners.shell_grid(geo["center"], geo["bound_radius"], *GRID)[:: P_LIS // n_lis][:n_lis]
    src = radiate.mc_sources(y, n, geo["total_area"], np.ones((len(ks), M_C4), complex),
                             np.tile(g8, (8, 1))[:, tri])
    radiate.radiate(src, ks, L)
    pairs += n_lis * M_C4 * len(ks)
    return pairs, time.perf_counter() - t0


class OraclePool:
    """The oracle on the host's cores: independent sample shares in separate processes."""

    def __init__(self):
        import multiprocessing as mp
        self.cores = len(os.sched_getaffinity(0))
        self.pool = mp.get_context("spawn").Pool(self.cores)

    def sample(self, rows_per_core=2, lis_per_core=8):
        jobs = [(c % N_GEO, [7 * c + r for r in range(rows_per_core)], lis_per_core) for c in range(self.cores)]
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_job, jobs)
        dt = time.perf_counter() - t0
        pairs = sum(r[0] for r in res)
        desc = (f"fp64 NumPy oracle, {self.cores} processes (one per host core): each takes one C4 geometry "
                f"(a1 + M = 2048 Philox samples), {rows_per_core} rows of the MC operator and right-hand side for "
                f"all 64 wavenumbers and the 64-mode radiation of the 2048 samples to {lis_per_core} of the 64^3 "
                f"listeners; pair-evals x wavenumbers / wall time")
        return pairs, dt, desc

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args):
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.destroy_process_group()
            return
    op = OraclePool()
    op.sample(1, 2)   # spawn + import
    for _ in range(args.warmup):
        op.sample(24, 16)
    tot_p, tot_t, desc = 0, 0.0, ""
    for _ in range(args.steps):
        p, t, desc = op.sample(24, 16)   # ~2-4 s per step
        tot_p += p
        tot_t += t
    op.close()
    val = tot_p / tot_t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": desc},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": op.cores, "kind": "oracle", "sample": desc}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def count_launches(sweep, torch, geo_ids):
    """Kernels of libnat launched during the step on `geo_ids` (torch.profiler / CUPTI)."""
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            sweep.run(geo_ids=geo_ids, n_workers=1)
            torch.cuda.synchronize()
        n_nat = 0
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                nm = e.name
                if "anonymous namespace" in nm or "nat::" in nm or "_GLOBAL__N_" in nm or "<unnamed>" in nm:
                    n_nat += 1
        return n_nat
    except Exception as ex:  # pragma: no cover
        print(f"[bench] launch count via profiler failed: {ex}", file=sys.stderr)
        return None


def mc_call_roofline(nat, torch, sweep, gi):
    """The BEM-MC estimator as ONE call (nat_mc_surface_pressure of geometry gi alone on the
    device, the library's single-call configuration): its binding roofline time (operator
    and right-hand-side pair-evaluations at R(n), from the kernel timer's per-launch buckets)
    over the call's device time (CUDA events, timer off).  In the sweep the same call overlaps
    other geometries; this is the latency view the verdict asked for."""
    h = sweep.host[gi]
    mesh, g = sweep.dmesh[gi], sweep.dg[gi]
    geo = nat.nat_mesh_prepare(mesh)
    plan = nat.McPlan(M_C4, N_K, "fp32", 200, "cuda")
    nat.single_call_tuning()
    try:
        def call():
            return nat.nat_mc_surface_pressure(mesh, geo, h["ks"], g, M_C4, seed=20250606, stream_id=gi, prec="fp32",
                                               tol=1e-6, plan=plan)
        call()
        torch.cuda.synchronize()
        nat.nat_kernel_timer_enable(True)
        call()
        torch.cuda.synchronize()
        t_roof = 0.0
        for cat, kind in ((nat.KTIMER_MC_OP, 1), (nat.KTIMER_MC_RHS, 2)):
            for n in range(1, 65):
                _, pairs, nl = nat.nat_kernel_timer_read(cat, n)
                if nl:
                    t_roof += pairs * sm_clk_per_pair(kind, n) / (SM_COUNT * MAX_MHZ * 1e6)
        nat.nat_kernel_timer_enable(False)
        ms = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, _, _, infos = call()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
    finally:
        nat.sweep_tuning()
    t = min(ms) * 1e-3
    return {"geometry": gi, "ms_per_call": 1e3 * t, "roofline_ms": 1e3 * t_roof, "frac": t_roof / t,
            "iterations_max": max(i["iters"] for i in infos), "solve_groups": 2,
            "note": "binding roofline of the call's pair work (operator + RHS at R(n)) / call time; the "
                    "rest is the 84-200-step Krylov chain (fused CGS2 step, epilogue, Givens)"}


def kernel_rooflines(nat, clk_mhz, traffic):
    """Per-category rooflines of the main pair kernels from the kernel timer's per-launch
    buckets (launches grouped by wavenumbers per pair): roofline time = pairs x binding
    SM-clocks per pair (sm_clk_per_pair) / (148 SM x clock)."""
    cats = {"mc_operator_kernel": (nat.KTIMER_MC_OP, 1, "radiate_f32x2_kernel<R,MB,1,NT> (a10 MC operator)"),
            "mc_rhs_kernel": (nat.KTIMER_MC_RHS, 2, "radiate_f32x2_kernel<R,MB,2,NT> (a9 MC right-hand side)"),
            "radiate_kernel": (nat.KTIMER_RADIATE, 0, "radiate_f32x2_kernel<R,MB,0,NT> (a11 radiation)")}
    out = {}
    for key, (cat, kind, name) in cats.items():
        sec_tot, pairs_tot, launches = nat.nat_kernel_timer_read(cat)
        if not launches:
            continue
        t_roof_max, t_roof_clk, mix = 0.0, 0.0, {}
        for n in range(1, 65):
            sec, pairs, nl = nat.nat_kernel_timer_read(cat, n)
            if not nl:
                continue
            c = sm_clk_per_pair(kind, n)
            t_roof_max += pairs * c / (SM_COUNT * MAX_MHZ * 1e6)
            t_roof_clk += pairs * c / (SM_COUNT * (clk_mhz or MAX_MHZ) * 1e6)
            mix[n] = nl
        achieved = pairs_tot / sec_tot / 1e9
        peak = pairs_tot / t_roof_max / 1e9
        out[key] = {"kernel": name, "bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gpair-evals/s",
                    "frac": t_roof_max / sec_tot, "frac_at_measured_clock": t_roof_clk / sec_tot,
                    "seconds": sec_tot, "launches": launches, "launch_mix_wavenumbers": mix,
                    "traffic": traffic.get(key), "peak_note":
                    "binding MUFU roofline of the minimal formulation per launch: (1 + 2n)/n MUFU per "
                    "pair-evaluation x wavenumber for n wavenumbers sharing rsqrt (16 MUFU/SM/clk, 148 SM, "
                    "1965 MHz max clock); FP32 (12 + 12n / 12 + 10n / 7 + 8n per pair)/n at 128 lanes never "
                    "binds (SURVEY.md §8(d), DESIGN.md §6)"}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    from paper_2506_06190_b200 import nat
    nat.sweep_tuning()
    nat.lib()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce_max_sum(ms, work):
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        w = torch.tensor([work], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(w, op=dist.ReduceOp.SUM)
        return t.item(), w.item()

    if args.workers <= 0:   # one rank's share at N = 8 is 8 geometries: all at once (measured 335 vs 340 ms)
        n_mine = len(geo_share(args.geometries, rank, world))
        args.workers = n_mine if n_mine <= 8 else 6
    sweep = Sweep(nat, torch, rank, world, args.workers, n_geo=args.geometries, e2e=not args.no_e2e)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def timed(steps, host_io=False):
        ev, tot = [], None
        barrier()
        for _ in range(steps):
            flush.fill_(1)   # L2 flush between timed steps (outside the step events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t_host = time.perf_counter()
            rec = sweep.run(host_io=host_io)
            e1.record()
            if sweep.verbose:
                hs = sorted(rec.pop("host_s", []), reverse=True)
                print(f"[bench] step host {time.perf_counter() - t_host:.3f} s, slowest geometries {hs[:4]}, "
                      f"median {hs[len(hs) // 2] if hs else None}", file=sys.stderr)
            ev.append((e0, e1))
            tot = merge(tot, rec)
        barrier()
        if os.environ.get("NAT_BENCH_VERBOSE"):
            print("[bench] step ms:", [round(a.elapsed_time(b), 1) for a, b in ev], file=sys.stderr)
        return sum(a.elapsed_time(b) for a, b in ev), tot

    for _ in range(max(3, args.warmup)):
        sweep.run()
    barrier()
    cs = ClockSampler(local)
    gc.collect()
    gc.disable()   # no collector pauses on the worker threads inside the timed steps
    with cs:
        ms, tot = timed(args.steps)
    gc.enable()
    clk = cs.summary()
    ms_max, pairs_all = allreduce_max_sum(ms, float(step_pairs(tot)))
    _, lis_all = allreduce_max_sum(0.0, float(tot["lis_pt_modes"]))
    value = pairs_all / (ms_max * 1e-3) / 1e9

    e2e = None
    if not args.no_e2e:
        sweep.run(host_io=True)   # warm the pinned paths
        gc.collect()
        gc.disable()
        ms_e, tot_e = timed(args.steps, host_io=True)
        gc.enable()
        ms_e_max, pe = allreduce_max_sum(ms_e, float(step_pairs(tot_e)))
        _, h2d = allreduce_max_sum(0.0, float(tot_e["h2d"]))
        _, d2h = allreduce_max_sum(0.0, float(tot_e["d2h"]))
        e2e = {"value": pe / (ms_e_max * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
               "ms_per_step": ms_e_max / args.steps,
               "note": "meshes + Neumann data H2D from pinned host and every 64 x 262,144 c128 field D2H to pinned "
                       "host (copy stream, double-buffered) inside the timed region, all ranks"}

    # per-kernel rooflines: a serialised pass (one worker, kernel timer on) over a few geometries
    sub = sweep.geo_ids[:4]
    nat.nat_kernel_timer_enable(True)
    cs2 = ClockSampler(local)
    with cs2:
        sweep.run(n_workers=1, geo_ids=sub, serial=True)
        torch.cuda.synchronize()
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    roofs = kernel_rooflines(nat, cs2.summary()["sm_mhz"], traffic)
    nat.nat_kernel_timer_enable(False)
    # the serialised pass's phase shares: dominant kernel by device time
    dom = max(roofs, key=lambda k: roofs[k]["seconds"]) if roofs else None
    roofline = dict(roofs[dom]) if dom else None
    if roofline:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sweep.run(n_workers=1, geo_ids=sub, serial=True)
        e1.record()
        torch.cuda.synchronize()
        roofline["share_of_serialised_step"] = roofline["seconds"] / (e0.elapsed_time(e1) * 1e-3)
        roofline["dominant"] = dom

    mc_call = mc_call_roofline(nat, torch, sweep, sweep.geo_ids[0])
    n_launch = None if args.no_profile_count else count_launches(sweep, torch, sweep.geo_ids[:1])

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        op = OraclePool()
        op.sample(1, 2)   # spawn + import warm-up
        p, t, desc = op.sample(rows_per_core=120, lis_per_core=80)   # ~10-20 s of host work
        op.close()
        cpu = {"value": p / t / 1e9, "unit": UNIT, "cores": op.cores, "kind": "oracle", "sample": desc, "seconds": t}
    K = args.steps
    its = tot["iters"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "geometries": args.geometries, "wavenumbers_per_geometry": N_K,
                   "M": M_C4, "listeners": P_LIS, "n_tri": sweep.n_tri,
                   "parallelism": f"geometries i mod {world}, {args.workers} worker streams per GPU",
                   "l2": "flushed (256 MB write) before every timed step"},
        "listener_pts_per_s": lis_all / (ms_max * 1e-3),
        "listener_pts_note": "listener points x wavenumbers radiated per second (whole step)",
        "pairs_per_step": pairs_all / K,
        "mc_gmres_iters": {"min": min(its), "mean": float(np.mean(its)), "max": max(its),
                           "systems": len(its) // K, "all_converged": bool(tot["converged"]),
                           "unconverged_systems": tot["unconverged"] // K,
                           "max_true_rel_residual": tot["max_rel_residual"],
                           "note": "tol 1e-6, 200 iterations (P:372); a system at the cap returns its best iterate, "
                                   "flagged, with its true residual (S:276)"},
        "roofline": roofline, "rooflines": roofs, "mc_call": mc_call,
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": (n_launch * len(sweep.geo_ids) * K) if n_launch else None,
        "gpu_launches_note": "libnat kernels of one geometry counted with torch.profiler (CUPTI) x geometries x steps",
        "clocks": clk,
        "secondary": None,
    }

    def emit(sec):
        if rank == 0:
            line["secondary"] = sec
            print(json.dumps(line), flush=True)

    secondary = None
    if not args.no_secondary:
        # the secondary lines run after the headline is final; a watchdog prints the headline
        # (and exits every rank) if they hang, e.g. in a collective at N > 1
        limit = float(os.environ.get("NAT_BENCH_SECONDARY_TIMEOUT", "300"))
        finished = threading.Event()
        partial = {}

        def watchdog():
            if not finished.wait(limit):
                emit(dict(partial, timeout=f"secondary lines unfinished after {limit:.0f} s"))
                os._exit(0)

        threading.Thread(target=watchdog, daemon=True).start()
        secondary = partial
        import bench_secondary as S
        comm = nat.Comm.from_torch_distributed() if world > 1 else None
        try:
            secondary["C2"] = S.run_c2(nat, torch, rank, world, comm, min(args.steps, 5), barrier, allreduce_max_sum)
        except Exception as ex:  # reported, not fatal: the headline is C4
            secondary["C2"] = {"error": repr(ex)}
        try:
            secondary["C3"] = S.run_c3(nat, torch, rank, world, min(args.steps, 5), barrier, allreduce_max_sum)
        except Exception as ex:
            secondary["C3"] = {"error": repr(ex)}
        try:
            pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
            secondary["NEXT4"] = S.run_nf(nat, torch, max(args.steps, 5),
                                          peaks=json.load(open(pk)) if os.path.exists(pk) else None)
        except Exception as ex:
            secondary["NEXT4"] = {"error": repr(ex)}
        finished.set()
    emit(secondary)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
