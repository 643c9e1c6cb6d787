"""Secondary bench lines (bench.py keys "secondary"): the C2 dense-BEM + BEM-MC step of
round 1 and the C3 modal BEM-MC solve.  Imported by bench.py only.

C2 (BASELINE.json configs[1]): oscillating-sphere dipole on the icosphere L5 (20,480
triangles) at ka in {0.5, 2, 8}: a1 mesh preparation, a12 32^3 listener grid, a2 near list,
per ka a4+a5 dense collocation assembly (fp32, c64 matrix) and a6+a7 GMRES (tol 1e-6), a11
radiation; BEM-MC on the same scene (M = 10,000) for the 3 wavenumbers and its
radiation.  At N > 1 the dense system is row-sharded (NCCL all-gather of the GMRES iterate)
and the MC wavenumbers are dealt to ranks (no collective).

C3 (configs[2]): the 49,664-triangle bowl, 32 modes (k a = 0.5 .. 8), M = 4096 uniform
samples, batched MC solve + fused 32-mode radiation to the 32^3 shell grid; at N > 1 each
rank takes the modes m with m mod N = rank.
"""
import os
import threading

import numpy as np

KAS = (0.5, 2.0, 8.0)
M_MC = 10000
GRID = (32, 32, 32)


def shard(n, rank, world):
    """Contiguous equal chunks (ceil) — the row ownership nat_bem_solve requires."""
    per = -(-n // world)
    return min(n, rank * per), min(n, (rank + 1) * per)


def mc_share(n_k, rank, world):
    return list(range(rank, n_k, world))


# ----------------------------------------------------------------------------------
# C2 step (round-1 headline, now a secondary line)
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
        self.order = os.environ.get("NAT_BENCH_ORDER", "multi")
        n_mat = len(KAS) if self.order in ("asm_first", "multi") else 1
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
            if self.order == "multi":
                # one far pass forms the three matrices (nat_bem_assemble_multi), then the solves
                self._ev("asm0", "m")
                nat.nat_bem_assemble_multi(self.mesh, geo, near, list(KAS), self.g, prec="fp32", A=self.A, lda=self.lda,
                                           rhs=self.b_bem)
                self._ev("asm1", "m")
                rows = self.r1 - self.r0
                with self.lock:
                    counts["far"] += rows * self.n * 3 * len(KAS)
                    counts["near"] += (self.nS * 448 + (near.nnz - self.nS) * 28) * len(KAS)
                    counts["self"] += rows * 48 * len(KAS)
                asm_ev.record(torch.cuda.current_stream())
                asm_done.set()
                for q in range(len(KAS)):
                    self._bem_one(q, geo, near, counts, assemble=False)
                    for grp in self.rad_groups:
                        if grp[-1] == q:
                            self._bem_radiate(geo, lis, grp, side)
                return
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
            if self.order in ("asm_first", "multi"):
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




def pairs_of(c):
    return c["far"] + c["near"] + c["self"] + c["rad"] + c["mc_rhs"] + c["mc_op"]


def load_c2_host():
    import nat_inputs as I
    m = I.icosphere(5)
    g = I.neumann_rigid_z(m)[None]
    return {"mesh": m, "g": g}


def run_c2(nat, torch, rank, world, comm, steps, barrier, allreduce_max_sum):
    """Timed C2 steps (chains serialised at N > 1: one communicator, one host thread).
    Returns the secondary-line dict."""
    os.environ.setdefault("NAT_BENCH_MC", "systems")   # MC wavenumbers dealt to ranks (no collective)
    step = Step(nat, torch, rank, world, comm, load_c2_host())
    overlap = world == 1
    step.overlap = overlap
    for _ in range(3):
        step.run()
    step.run(overlap=False)
    barrier()
    ms_steps, totals = [], None
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = step.run(overlap=overlap)
        e1.record()
        ms_steps.append((e0, e1))
        totals = c if totals is None else {k: totals[k] + v for k, v in c.items()}
    barrier()
    ms = sum(a.elapsed_time(b) for a, b in ms_steps)
    ms_max, pairs = allreduce_max_sum(ms, float(pairs_of(totals)))
    return {"workload": "C2: icosphere L5 (20,480 tri) dipole, ka in {0.5, 2, 8}: dense BEM (fp32 kernels, c64 "
                        "matrix, GMRES tol 1e-6) + BEM-MC (M = 10,000) + radiation to a 32^3 shell grid",
            "value": pairs / (ms_max * 1e-3) / 1e9, "unit": "Gpair-evals/s", "ms_per_step": ms_max / steps,
            "steps": steps, "overlap": overlap, "parallelism": f"rows (NCCL all-gather) x{world}" if world > 1 else "1 GPU",
            "gmres_iters": [it for _, it in sorted(totals["iters"][: len(KAS)])]}


def run_c3(nat, torch, rank, world, steps, barrier, allreduce_max_sum):
    import nat_inputs as I
    nat.single_call_tuning()   # one large solve at a time: the wide fused step, two solve groups
    m = I.bowl()
    mesh = nat.Mesh.from_numpy(m.v, m.t)
    ks_all = list(I.c3_wavenumbers())
    mine = [q for q in range(len(ks_all)) if q % world == rank]
    ks = [ks_all[q] for q in mine]
    g = torch.from_numpy(I.neumann_harmonics(m, 32)[mine]).cuda()
    M = 4096
    plan = nat.McPlan(M, len(ks), "fp32", 200, "cuda")
    P = GRID[0] * GRID[1] * GRID[2]
    rplan = nat.RadiatePlan(M, len(ks), P, "fp32", "cuda")
    out = torch.empty(len(ks), P, dtype=torch.complex128, device="cuda")
    lis = torch.empty(3, P, dtype=torch.float64, device="cuda")

    def one():
        geo = nat.nat_mesh_prepare(mesh)
        smp, stri, p, infos = nat.nat_mc_surface_pressure(mesh, geo, ks, g, M, seed=I.SEED, prec="fp32", plan=plan)
        src = nat.nat_mc_sources(smp, geo.total_area, p, nat.nat_mc_gather_neumann(g, stri), center=geo.center)
        nat.nat_listener_grid(geo.center, geo.bound_radius, *GRID, out=lis)
        nat.nat_radiate_field(src, ks, lis, "fp32", out=out, plan=rplan)
        return sum(M * (M - 1) * (1 + i["iters"]) for i in infos) + M * P * len(ks), [i["iters"] for i in infos]

    one()
    barrier()
    ev, pairs, iters = [], 0, None
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p_, iters = one()
        e1.record()
        ev.append((e0, e1))
        pairs += p_
    barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    ms_max, pairs_all = allreduce_max_sum(ms, float(pairs))
    return {"workload": "C3: bowl 49,664 tri, 32 modes (k a = 0.5..8), M = 4096 uniform samples, batched MC "
                        "solve (tol 1e-6) + fused 32-mode radiation to a 32^3 shell grid",
            "value": pairs_all / (ms_max * 1e-3) / 1e9, "unit": "Gpair-evals/s", "ms_per_step": ms_max / steps,
            "steps": steps, "parallelism": f"modes dealt x{world}" if world > 1 else "1 GPU",
            "mc_iters": iters}


def run_nf(nat, torch, steps, batch=262144, peaks=None):
    """NEXT-4 secondary line: training steps of the NAT neural field on
    C4-shaped samples — one config's 64^3 listener set per batch (normalised theta, phi, r;
    height, size, material), 8 outputs (|p| of the modes), synthetic smooth targets.
    Device time per step (CUDA events) and the tensor-core products' throughput
    (nat kernel timer: 2 M N K flops per product) against the measured bf16 peak."""
    import nat_inputs as I
    n_v, n_out = 3, 8
    shapes = nat.NeuralField.param_shapes(n_v, n_out)
    flat = torch.from_numpy(I.nf_init_params(shapes, 20250606, grid_scale=1e-4)).cuda()
    x = torch.from_numpy(I.nf_samples(batch, n_v, 20250607)).cuda()
    tgt = torch.stack([torch.sin(3 * x[:, 0] + q) * torch.cos(2 * x[:, 1]) * (1 + x[:, 3 + q % 3])
                       for q in range(n_out)], 1).contiguous()
    net = nat.NeuralField(n_v, n_out, flat, batch)
    for _ in range(3):
        net.train_step(x, tgt, 1e-3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss = net.train_step(x, tgt, 1e-3)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    nat.nat_kernel_timer_enable(True)
    net.train_step(x, tgt, 1e-3)
    sec, flops, nl = nat.nat_kernel_timer_read(nat.KTIMER_NF_GEMM)
    nat.nat_kernel_timer_enable(False)
    peak = (peaks or {}).get("bf16_tflops", 1590.0)
    hbm = (peaks or {}).get("hbm_gbs", 6650.0)
    # algorithmic HBM bytes of the 15 products per step (bf16 activations / gradients read
    # once and written once; weights negligible): forward, input gradients, weight gradients
    dims = [64, 128, 128, 128, 128, 16]
    fwd = sum(batch * 2 * (dims[q] + dims[q + 1]) for q in range(5))
    bwd_in = sum(batch * 2 * (dims[q + 1] + 2 * dims[q]) for q in range(5))
    bwd_w = sum(batch * 2 * (dims[q + 1] + dims[q]) for q in range(5))
    gemm_bytes = fwd + bwd_in + bwd_w
    return {"workload": f"NEXT-4 NAT neural field training step (hash grid 4 x 8..64, PE(6), 4 x 128 MLP, MSE, "
                        f"Adam), batch {batch} samples, 3 condition variables, 8 outputs, synthetic targets",
            "ms_per_step": ms, "samples_per_s": batch / (ms * 1e-3), "loss": float(loss.item()),
            "gemm": {"bound": "hbm", "bytes_per_step": gemm_bytes,
                     "achieved": gemm_bytes / sec / 1e9 if sec > 0 else None, "peak": hbm, "unit": "GB/s",
                     "frac": (gemm_bytes / sec / 1e9 / hbm) if sec > 0 else None,
                     "launches_per_step": nl, "gemm_ms_per_step": 1e3 * sec,
                     "arithmetic_intensity_flop_per_byte": flops / gemm_bytes,
                     "ridge_flop_per_byte": peak * 1e12 / (hbm * 1e9),
                     "peak_note": "MEASURED_PEAKS.json hbm_gbs; K <= 128 puts every layer product below the "
                                  "tensor/HBM ridge point, so the activations' traffic (read once, written once) "
                                  "is the binding roofline",
                     "tensor_view": {"bound": "tensor", "achieved": flops / sec / 1e12 if sec > 0 else None,
                                     "peak": peak, "unit": "TFLOP/s",
                                     "frac": (flops / sec / 1e12 / peak) if sec > 0 else None,
                                     "flops_per_step": flops,
                                     "peak_note": "MEASURED_PEAKS.json bf16_tflops (cuBLAS burst)"}}}
