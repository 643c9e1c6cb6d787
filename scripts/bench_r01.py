#!/usr/bin/env python3
"""bench.py — the NAT Helmholtz boundary-integral hot path on B200.

One *step* = one pass of every row of SURVEY.md §8(a) over the configuration the
metric is quoted on (BASELINE.json configs[1], "C2"): the oscillating-sphere dipole on
the icosphere L5 (20,480 triangles) at ka in {0.5, 2, 8}:

  a1 mesh preparation, a12 32^3 listener shell grid, a2 near list,
  per ka: a4+a5 dense collocation assembly (fp32, c64 matrix), a6+a7 GMRES
          (tol 1e-6, <= 200 it.), a11 radiation of the solution to the listeners;
  BEM-MC on the same scene (the paper's Table 2 pairing of BEM and BEM-MC, P:295-320;
  M = 10,000 samples as in P:320): a8 Philox samples, a9 RHS, a10 matrix-free operator
  inside batched GMRES for the 3 wavenumbers, a11 radiation of the MC solution.

Metric (BASELINE.json): Helmholtz kernel pair-evaluations/s (value, Gpair-evals/s) and
listener points/s, against the FP32-pipe roofline.  Multi-GPU (torchrun): the dense
system is row-sharded with an NCCL all-gather of the GMRES iterate, the listeners are
split by rank, the MC wavenumbers are dealt round-robin ("strong" scaling of one scene).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nat|reference]
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Helmholtz kernel Gpair-evals/s and listener pts/s vs FP32 roofline at 1/2/4/8 B200"
UNIT = "Gpair-evals/s"
KAS = (0.5, 2.0, 8.0)
M_MC = 10000
GRID = (32, 32, 32)
SM_COUNT, FP32_LANES, MAX_MHZ = 148, 128, 1965.0
# FP32-pipe roofline of one combined G + dG/dn_y pair (24 FP32-pipe instructions, 3 MUFU;
# DESIGN.md §5): 148 SM x 128 lanes x f / 24 = 16 MUFU/SM/clk x f / 3
R_PIPE = SM_COUNT * FP32_LANES * MAX_MHZ * 1e6 / 24.0
WORKLOAD = ("C2: oscillating-sphere dipole, icosphere L5 (20,480 tri), ka in {0.5, 2, 8}; dense "
            "BEM (fp32 kernels, c64 matrix, GMRES tol 1e-6) + BEM-MC (M = 10,000 uniform "
            "samples, tol 1e-6) + radiation of both solutions to a 32^3 shell grid (r = 1.5..3)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nat", choices=["nat", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile-count", action="store_true")
    ap.add_argument("--no-overlap", dest="overlap", action="store_false",
                    help="run the dense-BEM and BEM-MC chains one after the other")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(n, rank, world):
    """Contiguous equal chunks (ceil) — the row ownership nat_bem_solve requires."""
    per = -(-n // world)
    return min(n, rank * per), min(n, (rank + 1) * per)


def mc_share(n_k, rank, world):
    return list(range(rank, n_k, world))


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
            time.sleep(0.02)

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
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------------
# the GPU step
# ----------------------------------------------------------------------------------
class Step:
    def __init__(self, nat, torch, rank, world, comm, host):
        self.nat, self.torch, self.rank, self.world, self.comm = nat, torch, rank, world, comm
        self.comm_mc = None   # the BEM-MC chain's communicator (set by main at N > 1)
        self.host = host
        dev = torch.device("cuda")
        self.dev = dev
        m = host["mesh"]
        self.n = m.n_tri
        self.r0, self.r1 = shard(self.n, rank, world)
        P = GRID[0] * GRID[1] * GRID[2]
        self.P = P
        self.l0, self.l1 = shard(P, rank, world)
        # BEM-MC on > 1 rank: row-sharded (every rank owns sample rows of all the systems, one
        # all-gather per operator application) or, NAT_BENCH_MC=systems, whole
        # wavenumbers dealt round-robin (no collective)
        mc_mode = os.environ.get("NAT_BENCH_MC", "rows")   # rows | systems | rows_always (1-rank check)
        self.mc_sharded = (world > 1 and mc_mode == "rows") or mc_mode == "rows_always"
        self.mc_idx = list(range(len(KAS))) if self.mc_sharded else mc_share(len(KAS), rank, world)
        self.mc_r0, self.mc_r1 = shard(M_MC, rank, world) if self.mc_sharded else (0, M_MC)
        self.lock = threading.Lock()
        # device-resident inputs and buffers (allocated once, outside the timed region)
        self.mesh = nat.Mesh.from_numpy(m.v, m.t, device=dev)
        self.g = torch.from_numpy(host["g"]).to(dev)            # (1, n) dipole Neumann
        self.g_mc = self.g.expand(len(self.mc_idx), -1).contiguous() if self.mc_idx else None
        rows = self.r1 - self.r0
        self.lda = self.n + (self.n & 1)
        # dense-chain order: "interleave" (assembly + solve per wavenumber: one matrix, one
        # workspace) or "asm_first" (all assemblies, then the solves: one matrix per ka);
        # the three ka run one after the other in the dense-BEM chain (one NCCL communicator,
        # collectives issued in the same order on every rank).  NAT_BENCH_ORDER overrides.
        self.order = os.environ.get("NAT_BENCH_ORDER", "interleave")
        n_mat = len(KAS) if self.order == "asm_first" else 1
        mats = [torch.empty(rows, self.lda, dtype=torch.complex64, device=dev) for _ in range(n_mat)]
        wss = [nat._ws(nat.lib().nat_bem_solve_workspace(nat.NAT_FP32, self.n, rows, 200), dev) for _ in range(n_mat)]
        self.A = [mats[q % n_mat] for q in range(len(KAS))]
        self.solve_ws = [wss[q % n_mat] for q in range(len(KAS))]
        self.S_bem = 3 * self.n
        self.n_lis = self.l1 - self.l0
        # BEM radiation groups: the solutions of each group of wavenumbers radiate in one
        # fused launch as soon as the group's last solve is done (NAT_BENCH_RADGROUPS,
        # e.g. "012" = one launch after the last solve, "01,2", "0,1,2")
        self.rad_groups = [[int(c) for c in g] for g in os.environ.get("NAT_BENCH_RADGROUPS", "012").split(",")]
        self.rad_plan_bem = {len(g): nat.RadiatePlan(self.S_bem, len(g), self.n_lis, "fp32", dev)
                             for g in self.rad_groups}
        self.out_bem = torch.empty(len(KAS), self.n_lis, dtype=torch.complex128, device=dev)
        self.x_bem = torch.empty(len(KAS), self.n, dtype=torch.complex128, device=dev)
        self.b_bem = torch.empty(len(KAS), 1, self.r1 - self.r0, dtype=torch.complex128, device=dev)

        self.g3 = self.g.expand(len(KAS), -1).contiguous()
        if self.mc_idx:
            self.mc_plan = nat.McPlan(M_MC, len(self.mc_idx), "fp32", 200, dev)
            if self.mc_sharded:
                self.mc_shard_ws = nat._ws(nat.lib().nat_mc_sharded_workspace(nat.NAT_FP32, M_MC, len(self.mc_idx),
                                                                              200, world), dev)
            self.rad_plan_mc = nat.RadiatePlan(M_MC, len(self.mc_idx), self.n_lis, "fp32", dev)
            self.out_mc = torch.empty(len(self.mc_idx), self.n_lis, dtype=torch.complex128, device=dev)
        self.ev = {}
        self.overlap = True
        # the MC chain gets the high-priority stream: its FP32/MUFU-bound launches run at full
        # rate while the dense-BEM chains (HBM-bound GEMV) fill the remaining issue slots
        prio = os.environ.get("NAT_BENCH_PRIO", "mc")
        self.s_bem = torch.cuda.Stream(priority=-1 if prio == "bem" else 0)
        self.s_mc = torch.cuda.Stream(priority=-1 if prio == "mc" else 0)
        self.s_rad = torch.cuda.Stream()

    def _ev(self, name, tag=""):
        """Event on the current stream; `tag` keeps the start/end events of concurrent
        chains apart (phase spans pair events with the same tag)."""
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        with self.lock:
            self.ev.setdefault(name, {}).setdefault(tag, []).append(e)

    def run(self, host_inputs=False, overlap=None):
        """One step.  host_inputs=True: the step's inputs (mesh, Neumann data) are copied
        from pinned host memory and the results read back (the e2e measurement).
        overlap=True: the dense-BEM chain (assembly, HBM-bound GEMV solve, radiation) and
        the BEM-MC chain (FP32/MUFU-bound operators, radiation) run concurrently on two
        streams from two host threads (the C calls release the GIL), so the compute-bound MC
        kernels fill the SMs the GEMV leaves idle."""
        nat, torch = self.nat, self.torch
        overlap = self.overlap if overlap is None else overlap
        mesh, g = self.mesh, self.g
        if host_inputs:
            hv, ht, hg = self.host["pinned"]
            mesh.vxyz.copy_(hv, non_blocking=True)
            mesh.tri.copy_(ht, non_blocking=True)
            g.copy_(hg, non_blocking=True)
            self.g3.copy_(g.expand(len(KAS), -1))
            if self.g_mc is not None:
                self.g_mc.copy_(g.expand(len(self.mc_idx), -1))
        self._ev("geom0")
        geo = nat.nat_mesh_prepare(mesh)                                              # a1
        lis = nat.nat_listener_grid((0.0, 0.0, 0.0), 1.0, *GRID, device=self.dev)    # a12
        if self.world > 1:
            lis = lis[:, self.l0:self.l1].contiguous()
        self._ev("geom1")
        # a2 before the fork: only the dense-BEM chain (the critical path) needs it, and it
        # runs fastest with the GPU to itself
        self._ev("near0")
        near = nat.nat_bem_near_list(mesh, geo, self.r0, self.r1)                   # a2
        self._ev("near1")
        counts = dict(far=0, near=0, self=0, rad=0, mc_rhs=0, mc_op=0, gemv_bytes=0, gemv_s=0.0,
                      mc_op_s=0.0, iters=[], mc_iters=[])

        if not hasattr(self, "nS"):   # class counts for the pair accounting (first step only)
            self.nS = int((near.cls == 1).sum().item())

        asm_done = threading.Event()   # host-side: the dense chain has enqueued its assemblies
        asm_ev = torch.cuda.Event()

        def bem_all(side=None):
            if self.order == "asm_first":
                # all assemblies first (FP32/MUFU-bound), then the HBM-bound GMRES solves,
                # which the MC chain's FP32/MUFU-bound operators overlap
                for q in range(len(KAS)):
                    self._bem_one(q, geo, near, counts, solve=False)
                asm_ev.record(torch.cuda.current_stream())
                asm_done.set()
                for q in range(len(KAS)):
                    self._bem_one(q, geo, near, counts, assemble=False)
                    for grp in self.rad_groups:
                        if grp[-1] == q:
                            self._bem_radiate(geo, lis, grp, side)
                return
            for q in range(len(KAS)):
                self._bem_one(q, geo, near, counts)
                for grp in self.rad_groups:
                    if grp[-1] == q:
                        self._bem_radiate(geo, lis, grp, side)

        def mc_after_asm(*a):
            if self.order == "asm_first":
                asm_done.wait()
                torch.cuda.current_stream().wait_event(asm_ev)
            self._mc_chain(*a)

        if not overlap:
            bem_all()
            if self.mc_idx:
                self._mc_chain(geo, lis, counts)
        else:
            cur = torch.cuda.current_stream()
            ready = torch.cuda.Event()
            ready.record(cur)
            err = []

            def worker(stream, fn, *a):
                try:
                    with torch.cuda.stream(stream):
                        stream.wait_event(ready)
                        fn(*a)
                except BaseException as ex:  # re-raised on the main thread
                    err.append(ex)

            ths = [threading.Thread(target=worker, args=(self.s_bem, bem_all, self.s_rad))]
            if self.mc_idx:
                ths.append(threading.Thread(target=worker, args=(self.s_mc, mc_after_asm, geo, lis, counts)))
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            if err:
                raise err[0]
            cur.wait_stream(self.s_bem)
            cur.wait_stream(self.s_rad)
            cur.wait_stream(self.s_mc)
        if host_inputs:
            hb, hm = self.host["out_pinned"]
            hb.copy_(self.out_bem, non_blocking=True)
            if self.mc_idx:
                hm[: self.out_mc.shape[0]].copy_(self.out_mc, non_blocking=True)
        return counts

    def _bem_one(self, q, geo, near, counts, assemble=True, solve=True):
        """a4-a7 for KAS[q] (row-sharded across ranks)."""
        nat = self.nat
        mesh, g = self.mesh, self.g
        nS, nN = self.nS, near.nnz - self.nS
        rows = self.r1 - self.r0
        tag = str(q)
        if assemble:
            self._ev("asm0", tag)
            A, b = nat.nat_bem_assemble(mesh, geo, near, KAS[q], g, prec="fp32", A=self.A[q], lda=self.lda,
                                        rhs=self.b_bem[q])                                          # a4+a5
            self._ev("asm1", tag)
            with self.lock:
                counts["far"] += rows * self.n * 3
                counts["near"] += nS * 448 + nN * 28
                counts["self"] += rows * 48
        if not solve:
            return
        self._ev("solve0", tag)
        _, info = nat.nat_bem_solve(self.A[q], self.b_bem[q][0], self.n, self.r0, self.comm, tol=1e-6, max_iter=200,
                                    ws=self.solve_ws[q], out=self.x_bem[q])                       # a6+a7
        self._ev("solve1", tag)
        with self.lock:
            counts["rad"] += self.S_bem * self.n_lis
            counts["gemv_bytes"] += info["iters"] * rows * self.lda * 8
            counts["gemv_s"] += info["t_matvec_s"]
            counts["iters"].append((q, info["iters"]))

    def _bem_radiate(self, geo, lis, grp, side=None):
        """a11 for the solutions of the wavenumbers in grp (contiguous indices), one fused
        launch (shared r, 1/r, d.n per pair).  side: a stream that waits for the solves
        and runs the radiation beside the next assembly / solve."""
        nat, torch = self.nat, self.torch
        a, b = grp[0], grp[-1] + 1

        def go():
            src = nat.nat_bem_sources(self.mesh, geo, self.x_bem[a:b], self.g3[a:b])
            self._ev("rad0", str(a))
            nat.nat_radiate_field(src, list(KAS[a:b]), lis, "fp32", out=self.out_bem[a:b],
                                  plan=self.rad_plan_bem[b - a])
            self._ev("rad1", str(a))

        if side is None:
            go()
        else:
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                go()

    def _mc_chain(self, geo, lis, counts):
        """a8-a10 (batched over the rank's wavenumbers), then a11 of the MC solution."""
        nat = self.nat
        ks = [KAS[i] for i in self.mc_idx]
        self._ev("mc0")
        if self.mc_sharded:
            smp, stri, p, infos = nat.nat_mc_surface_pressure_sharded(
                self.mesh, geo, ks, self.g_mc, M_MC, self.comm_mc, seed=20250606, stream_id=0, prec="fp32", tol=1e-6,
                ws=self.mc_shard_ws)                                                                 # a8-a10, rows
        else:
            smp, stri, p, infos = nat.nat_mc_surface_pressure(self.mesh, geo, ks, self.g_mc, M_MC, seed=20250606,
                                                              stream_id=0, prec="fp32", tol=1e-6,
                                                              plan=self.mc_plan)                # a8-a10
        self._ev("mc1")
        gs = nat.nat_mc_gather_neumann(self.g_mc, stri)
        src = nat.nat_mc_sources(smp, geo.total_area, p, gs)
        self._ev("radmc0")
        nat.nat_radiate_field(src, ks, lis, "fp32", out=self.out_mc, plan=self.rad_plan_mc)          # a11
        self._ev("radmc1")
        with self.lock:
            counts["mc_op_s"] += infos[0]["t_matvec_s"] if infos else 0.0   # one batch: shared
            mc_rows = self.mc_r1 - self.mc_r0   # this rank's operator rows
            for inf in infos:
                counts["mc_rhs"] += mc_rows * (M_MC - 1)
                counts["mc_op"] += inf["iters"] * mc_rows * (M_MC - 1)
                counts["mc_iters"].append(inf["iters"])
            counts["rad"] += M_MC * self.n_lis * len(ks)

    def phase_ms(self):
        """Device time per phase, summed over the recorded steps (call after sync)."""
        def span(a, b):
            ea, eb = self.ev.get(a, {}), self.ev.get(b, {})
            return sum(x.elapsed_time(y) for t in ea for x, y in zip(ea[t], eb.get(t, [])))
        return {"geometry": span("geom0", "geom1"), "near_list": span("near0", "near1"),
                "assembly": span("asm0", "asm1"),
                "bem_solve": span("solve0", "solve1"), "radiate_bem": span("rad0", "rad1"),
                "mc_solve": span("mc0", "mc1"), "radiate_mc": span("radmc0", "radmc1")}


def pairs_of(c):
    return c["far"] + c["near"] + c["self"] + c["rad"] + c["mc_rhs"] + c["mc_op"]


# ----------------------------------------------------------------------------------
# oracle timing (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------------
def oracle_sample(host, scale=1):
    """Times the fp64 oracle, as it stands, on a bounded sample of the same workload
    (scale 1: 4 full rows of the C2 dense assembly at ka = 8 with far + near + self rules,
    radiation of the 61,440 BEM sources to 64 listeners, 8 rows of the BEM-MC operator and
    RHS at M = 10,000; every count is multiplied by ``scale``).
    Returns (pair-evals, seconds, description)."""
    from oracle import bem, geometry, kernel, listeners, mc, nearlist, radiate
    m = host["mesh"]
    t0 = time.perf_counter()
    geo = geometry.mesh_prepare(m.v, m.t)
    rows = np.linspace(0, m.n_tri - 1, 4 * scale).astype(int)
    A, b = bem.assemble(m.v, m.t, geo, 8.0, host["g"], rows=rows)
    rp, col, cls = nearlist.near_list(m.t, geo["centroid"], geo["diam"], rows=rows)
    n_pairs = len(rows) * m.n_tri * 3 + int((cls == 1).sum()) * 448 + int((cls == 2).sum()) * 28 + len(rows) * 48
    x = np.ones(m.n_tri, dtype=complex)
    src = radiate.bem_sources(m.v, m.t, geo, x[None], host["g"])
    nl = 64 * scale
    L = listeners.shell_grid(np.zeros(3), 1.0, *GRID)[:: (GRID[0] * GRID[1] * GRID[2]) // nl][:nl]
    radiate.radiate(src, [8.0], L)
    n_pairs += nl * src[0].shape[0]
    y, n, tri = mc.sample_uniform(m.v, m.t, geo, M_MC, 20250606, 0)
    eps = mc.default_eps(geo["total_area"], M_MC)
    w = mc.weight(geo["total_area"], M_MC, eps)
    g = host["g"][0][tri]
    p = np.ones(M_MC, dtype=complex)
    for i in range(8 * scale):
        j = np.arange(M_MC) != i
        _ = 0.5 * p[i] - w * np.sum(kernel.green_dn_y(y[i], y[j], n[j], 8.0) * p[j])
        _ = -w * np.sum(kernel.green(y[i], y[j], 8.0) * g[j]) - 0.5 * eps * g[i]
        n_pairs += 2 * (M_MC - 1)
    dt = time.perf_counter() - t0
    desc = (f"fp64 NumPy oracle on a bounded sample of the C2 step: {len(rows)} full rows of the dense "
            f"assembly at ka=8 (far+near+self rules), radiation of 61,440 BEM sources to {nl} "
            f"listeners, {8 * scale} rows of the BEM-MC operator and RHS (M=10,000); pair-evals/s")
    return n_pairs, dt, desc


def oracle_cores():
    # NumPy ufuncs (the oracle's hot loops) run on one thread.
    return 1


def load_host():
    import nat_inputs as I
    m = I.icosphere(5)
    g = I.neumann_rigid_z(m)[None]
    return {"mesh": m, "g": g}


def run_reference(args):
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.destroy_process_group()
            return
    host = load_host()
    for _ in range(args.warmup):
        oracle_sample(host)
    tot_p, tot_t = 0, 0.0
    for _ in range(args.steps):
        p, t, desc = oracle_sample(host)
        tot_p += p
        tot_t += t
    val = tot_p / tot_t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": desc},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle_cores(), "kind": "oracle",
                             "sample": desc}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def count_launches(step, torch):
    """Kernels of libnat launched during one step (torch.profiler / CUPTI)."""
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step.run()
            torch.cuda.synchronize()
        n_all, n_nat = 0, 0
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                n_all += 1
                nm = e.name
                if "anonymous namespace" in nm or "nat::" in nm or "_GLOBAL__N_" in nm:
                    n_nat += 1
        return n_nat, n_all
    except Exception as ex:  # pragma: no cover
        print(f"[bench] launch count via profiler failed: {ex}", file=sys.stderr)
        return None, None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    from paper_2506_06190_b200 import nat
    nat.lib()
    comm = comm_mc = None
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
        comm = nat.Comm.from_torch_distributed()
        # the BEM-MC chain runs beside the dense chain from another host thread: its
        # all-gathers get their own communicator, so each communicator sees its collectives
        # in the same order on every rank (two threads interleaving on one would deadlock)
        comm_mc = nat.Comm.from_torch_distributed()
    host = load_host()
    step = Step(nat, torch, rank, world, comm, host)
    step.comm_mc = comm_mc
    step.overlap = args.overlap
    # pinned host copies for the e2e measurement
    m = host["mesh"]
    hv = torch.from_numpy(np.ascontiguousarray(m.v.T)).pin_memory()
    ht = torch.from_numpy(np.ascontiguousarray(m.t.T.astype(np.int32))).pin_memory()
    hg = torch.from_numpy(host["g"]).pin_memory()
    host["pinned"] = (hv, ht, hg)
    host["out_pinned"] = (torch.empty(step.out_bem.shape, dtype=torch.complex128).pin_memory(),
                          torch.empty((len(KAS), step.n_lis), dtype=torch.complex128).pin_memory())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        step.run()
    if args.overlap:
        step.run(overlap=False)   # the serialised steps below allocate on the default stream
    barrier()

    def timed(overlap):
        """K steps bracketed by barrier + synchronize; returns (ms, totals, phases)."""
        step.ev = {}
        totals, ms_steps = None, []
        barrier()
        for _ in range(args.steps):
            flush.fill_(1)   # L2 flush between timed iterations (outside the step events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            c = step.run(overlap=overlap)
            e1.record()
            ms_steps.append((e0, e1))
            if totals is None:
                totals = {k: (v if not isinstance(v, list) else list(v)) for k, v in c.items()}
            else:
                for k, v in c.items():
                    totals[k] = totals[k] + v
        barrier()
        return sum(a.elapsed_time(b) for a, b in ms_steps), totals, step.phase_ms()

    cs = ClockSampler(local)
    with cs:
        ms, totals, _ = timed(args.overlap)
    # per-kernel rooflines and phase times come from the same steps with the two chains
    # serialised (overlapped kernels share the SMs, so their spans would not be per-kernel)
    ms_seq, totals_seq, phases = timed(False) if args.overlap else (ms, totals, step.phase_ms())
    # per-kernel device time: CUDA events on the launching stream around each main kernel
    # (libnat's kernel timer), K more serialised steps so the passes above stay unperturbed
    nat.nat_kernel_timer_enable(True)
    timed(False)
    ktimes = {name: nat.nat_kernel_timer_read(cat) for name, cat in
              (("mc_op", nat.KTIMER_MC_OP), ("mc_rhs", nat.KTIMER_MC_RHS), ("radiate", nat.KTIMER_RADIATE),
               ("far", nat.KTIMER_FAR))}
    nat.nat_kernel_timer_enable(False)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    pairs_t = torch.tensor([float(pairs_of(totals)), float(totals["rad"])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(pairs_t, op=dist.ReduceOp.SUM)
    ms_max = ms_t.item()
    pairs_all, rad_pairs_all = pairs_t.tolist()
    value = pairs_all / (ms_max * 1e-3) / 1e9

    # e2e: same steps with host inputs / outputs (pinned) inside the timed region
    e2e = None
    if not args.no_e2e:
        step.ev = {}
        barrier()
        ev = []
        p_e2e = 0
        for _ in range(args.steps):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            c = step.run(host_inputs=True)
            e1.record()
            ev.append((e0, e1))
            p_e2e += pairs_of(c)
        barrier()
        ms_e = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device="cuda")
        pe = torch.tensor([float(p_e2e)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ms_e, op=dist.ReduceOp.MAX)
            dist.all_reduce(pe, op=dist.ReduceOp.SUM)
        h2d = hv.numel() * 8 + ht.numel() * 4 + hg.numel() * 16
        d2h = step.out_bem.numel() * 16 + (step.out_mc.numel() * 16 if step.mc_idx else 0)
        e2e = {"value": pe.item() / (ms_e.item() * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    n_nat, n_all = (None, None) if args.no_profile_count else count_launches(step, torch)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    clk = cs.summary()
    # rooflines of the kernels (achieved / measured-or-derived peak); DESIGN.md §5
    t_rad = (phases["radiate_bem"] + phases["radiate_mc"]) * 1e-3
    t_asm = phases["assembly"] * 1e-3
    t_mc = phases["mc_solve"] * 1e-3
    t_gemv = totals_seq["gemv_s"]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    hbm = peaks.get("hbm_gbs", 6650.0)
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))

    def alu(name, pairs, t, tkey):
        a = pairs / t / 1e9 if t > 0 else 0.0
        return {"kernel": name, "bound": "alu", "achieved": a, "peak": R_PIPE / 1e9, "unit": "Gpair-evals/s",
                "frac": a / (R_PIPE / 1e9), "traffic": traffic.get(tkey), "traffic_kernel": tkey,
                "traffic_note": "dram read+write bytes per launch, ncu --set full (profiles/traffic.json)",
                "peak_note": "FP32-pipe roofline: 148 SM x 128 lanes x 1965 MHz / 24 instr per combined "
                             "G+dG pair (= 16 MUFU/SM/clk / 3); derived, DESIGN.md §5",
                "frac_at_measured_clock": (a / (R_PIPE / 1e9) * MAX_MHZ / clk["sm_mhz"]) if clk["sm_mhz"] else None}

    roof = {
        "radiate": alu("nat_radiate_field (stage + radiate_f32x2_kernel + split reduce)", totals_seq["rad"], t_rad,
                       "radiate_f32x2_kernel<2, 3, 0, 256>"),
        "bem_assembly": alu("nat_bem_assemble (far_kernel_x2 + near/self kernels)",
                            totals_seq["far"] + totals_seq["near"] + totals_seq["self"], t_asm, "far_kernel_x2<3, 1, 0, 1>"),
        "mc_solve": alu("MC solve phase (a8-a10: samples, close pairs, RHS, operator, GMRES)",
                        totals_seq["mc_op"] + totals_seq["mc_rhs"], t_mc, None),
        "mc_operator": alu("MC operator application (stage + radiate_f32x2_kernel<R,MB,1,NT> + mc_finish_kernel)",
                           totals_seq["mc_op"], totals_seq["mc_op_s"], "radiate_f32x2_kernel<2, 3, 1, 256>"),
        "gemv": {"kernel": "gemv_c64_kernel", "bound": "hbm",
                 "achieved": totals_seq["gemv_bytes"] / t_gemv / 1e9 if t_gemv > 0 else 0.0,
                 "peak": hbm, "unit": "GB/s",
                 "frac": (totals_seq["gemv_bytes"] / t_gemv / 1e9 / hbm) if t_gemv > 0 else 0.0,
                 "traffic": traffic.get("gemv_c64_kernel"), "traffic_kernel": "gemv_c64_kernel",
                 "peak_note": "measured HBM copy bandwidth, MEASURED_PEAKS.json"},
    }
    # single kernels, timed per launch with CUDA events on their stream (libnat kernel timer)
    kt_names = {"mc_op": ("radiate_f32x2_kernel<R,MB,1,NT> (a10 MC operator main kernel)",
                          "radiate_f32x2_kernel<2, 3, 1, 256>"),
                "radiate": ("radiate_f32x2_kernel<R,MB,0,NT> (a11 radiation main kernel)",
                            "radiate_f32x2_kernel<2, 3, 0, 256>"),
                "far": ("far_kernel_x2<3,1> (a4 far assembly + fused RHS, 8 B store per entry)", "far_kernel_x2<3, 1, 0, 1>"),
                "mc_rhs": ("radiate_f32x2_kernel<R,MB,2,NT> (a9 MC right-hand side main kernel)",
                           "radiate_f32x2_kernel<2, 3, 2, 256>")}
    for key, (name, tkey) in kt_names.items():
        sec, pairs_k, nl = ktimes[key]
        if nl:
            r = alu(name, pairs_k, sec, tkey)
            r["launches_per_step"] = nl / args.steps
            r["ms_per_step"] = 1e3 * sec / args.steps
            roof[key + "_kernel"] = r
    # dominant KERNEL by device time per step (single kernels; the GEMV is one kernel per call)
    share = {k + "_kernel": ktimes[k][0] for k in kt_names if ktimes[k][2]}
    share["gemv"] = t_gemv
    dom = max(share, key=share.get)
    roofline = dict(roof[dom])
    roofline["share_of_step"] = share[dom] / (ms_seq * 1e-3)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        p, t, desc = oracle_sample(host, scale=16)   # ~10-20 s of host work
        cpu = {"value": p / t / 1e9, "unit": UNIT, "cores": oracle_cores(), "kind": "oracle", "sample": desc,
               "seconds": t}
    K = args.steps
    per_step_launch = n_nat
    bsm_meas = (phases["assembly"] + phases["bem_solve"]) * 1e-3 / (K * len(KAS))
    bsm_roof = ((totals_seq["far"] + totals_seq["near"] + totals_seq["self"]) / R_PIPE
                + totals_seq["gemv_bytes"] / (hbm * 1e9)) / (K * len(KAS))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_tri": step.n, "listeners": step.P, "M_mc": M_MC, "ka": list(KAS),
                   "parallelism": f"rows/listeners x{world}", "l2": "flushed (256 MB write) before every timed step"},
        "listener_pts_per_s": (K * step.P * (len(KAS) + len(KAS))) / (ms_max * 1e-3) if world == 1 else None,
        "radiate_listener_pts_per_s": (step.n_lis * (len(KAS) + len(step.mc_idx)) * K) / t_rad if t_rad > 0 else None,
        "pairs_per_step": pairs_all / K,
        # BEM solve seconds per mode against its roofline
        # (a4 + a5 evaluations / R_pipe + the GEMV bytes of its iterations / HBM copy bandwidth)
        "bem_s_per_mode": {
            "measured": bsm_meas, "roofline": bsm_roof, "frac": bsm_roof / bsm_meas if bsm_meas > 0 else None,
            "note": "per wavenumber: assembly + GMRES (serialised pass); roofline = pair-evals / R_pipe + "
                    "matrix bytes streamed / measured HBM copy bandwidth"},
        # radiation listener points (x wavenumbers, BEM 61,440 + MC 10,000 sources) per second
        # at the pair roofline: the same points / (their pair-evaluations / R_pipe)
        "radiate_listener_pts_roofline_per_s": (step.n_lis * (len(KAS) + len(step.mc_idx)) * K) * R_PIPE
                                               / totals_seq["rad"] if totals_seq["rad"] else None,
        "phase_ms_per_step": {k: v / K for k, v in phases.items()},
        "phase_note": ("phases and rooflines from K more steps with the two chains serialised "
                       f"({ms_seq / K:.3f} ms/step); value/ms_per_step from the overlapped steps")
        if args.overlap else "chains serialised (--no-overlap)",
        "overlap": bool(args.overlap),
        "gmres_iters": [it for _, it in sorted(totals["iters"][: len(KAS)])], "mc_gmres_iters": totals["mc_iters"][: len(step.mc_idx)],
        "roofline": roofline, "rooflines": roof,
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": (per_step_launch * K) if per_step_launch is not None else None,
        "gpu_launches_note": "libnat kernels per step counted with torch.profiler (CUPTI) x steps",
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
