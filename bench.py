#!/usr/bin/env python
"""Benchmark of the GN Hessian-matvec hot path (BASELINE.json north_star).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--size 256] [--degree 3]

One step = one Gauss-Newton Hessian matvec (optim.hpp:115-137, Transpose
adjoint, gradient cache on) at the SYN linearisation point v = 0.5 v_syn,
vt = -g, nt = 4, cubic, beta = 1e-3, fp32 on device.
N = 1: the 256^3 configuration (BASELINE.json configs[1]). N > 1: weak
scaling at 256^3 voxels per GPU, slab-decomposed along x1
(512x256x256 @2, 512x512x256 @4, 512^3 @8); --size 512 gives the 512^3-per-GPU
family up to 1024^3 on 8 GPUs.

Metric: matvec throughput in Mvox*matvec/s (grid points x matvecs / s),
whole job. Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GN Hessian matvec throughput (SYN, nt=4, cubic, H1, beta=1e-3)"
UNIT = "Mvox*matvec/s"
BETA = 1e-3
NT = 4


def weak_grid(n, N):
    """Per-GPU work fixed: double x1, then x2, then x3 (slab axis first)."""
    dims = [n, n, n]
    k, a = N, 0
    while k > 1:
        dims[a % 3] *= 2
        k //= 2
        a += 1
    return tuple(dims)


def bytes_per_voxel(nt):
    """Fused-minimum HBM bytes per voxel of the GN matvec, SURVEY.md §8(d):
    inc-state 24 + 52 nt, transpose + final 40 + 64 nt, spectral symbol 24
    (88 + 116 nt; 552 at nt = 4). The roofline denominator for matvec_gbs."""
    return 88 + 116 * nt


def bytes_per_voxel_ours(nt):
    """What our kernels move per voxel: inc-state pre-pass
    12 (nt + 1) + 16 + 4 nt, nt steps x 24, nt scatter sweeps x 28, assembly
    16 (nt + 1) + 24, separable regulariser 3 x (8 + 12 + 12)."""
    return 12 * (nt + 1) + 16 + 4 * nt + 24 * nt + 28 * nt + 16 * (nt + 1) + 24 + 3 * 32


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, start: bool):
        """Bracket the timed region: summary() prefers samples inside it."""
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        inside = [ln for t, ln in self.lines if t0 is not None and t1 is not None and t0 <= t <= t1 + 0.02]
        use = inside or [ln for _, ln in self.lines]
        for ln in use:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "samples_in_timed_region": len(inside),
                "interval_ms": 20}


def measured_peak():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        try:
            with open(p) as f:
                return float(json.load(f)["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    --set full summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def ncu_smem_wavefronts():
    """Per-launch shared-memory wavefronts (ncu l1tex__data_pipe_lsu_wavefronts_
    mem_shared) of the SL kernels from profiles/smem_wavefronts.json, or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "smem_wavefronts.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# --------------------------------------------------------------- CPU legs ----

def _ref_session(n):
    """The UNMODIFIED reference (oracle/_ref) at the bench linearisation point
    (SYN, v = 0.5 v_syn, vt = -g). Returns (session, vt)."""
    from oracle import ref
    m0, v, m1 = ref.syn(n, NT, 3)
    s = ref.Session(m0, m1, 0.5 * v, BETA, ref.Config(continuation=False, beta_target=BETA))
    return s, -s.gradient()


def cpu_reference_sample(n=256, matvecs=1):
    """`matvecs` GN matvecs of the compiled reference (fp64; single-threaded:
    it has no OpenMP or threads) on the host at the benchmark grid. Returns
    (Mvox*matvec/s, seconds, kind, sample, reference KernelTimers per matvec)."""
    from oracle import ref
    if ref.available():
        s, vt = _ref_session(n)
        t_before = s.timers()
        t0 = time.perf_counter()
        for _ in range(matvecs):
            s.matvec(vt)
        dt = time.perf_counter() - t0
        t_after = s.timers()
        timers = {k: (t_after[k] - t_before[k]) / matvecs for k in t_after}
        return n ** 3 * matvecs / dt / 1e6, dt, "reference", \
            f"{matvecs} GN matvec(s) of the compiled reference at {n}^3 (fp64, 1 thread)", timers
    from oracle import vreg_np as O
    n = min(n, 64)
    m0 = O.syn_template((n,) * 3)
    v = O.syn_velocity((n,) * 3)
    fwd, _ = O.characteristics(v, NT)
    m1 = O.solve_state(fwd, m0, NT)[-1]
    L = O.Linearization(m0, m1, 0.5 * v, BETA)
    t0 = time.perf_counter()
    for _ in range(matvecs):
        L.matvec(-L.g)
    dt = time.perf_counter() - t0
    return n ** 3 * matvecs / dt / 1e6, dt, "port", \
        f"{matvecs} GN matvec(s) of the numpy restatement at {n}^3 (fp64)", None


def run_reference(args):
    """Reference arm: the compiled reference's own GN matvec
    (detail::hessian_matvec_with, optim.hpp:115-137) on the host, one matvec
    of the benchmark grid per step (the same config as our arm, N = 1)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    nx, ny, nz = (args.size,) * 3 if args.gpus == 1 else weak_grid(args.size, args.gpus)
    n = args.size
    same = args.gpus == 1
    if ref.available():
        s, vt = _ref_session(n)
        for _ in range(args.warmup):
            s.matvec(vt)
        t_before = s.timers()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s.matvec(vt)
        dt = time.perf_counter() - t0
        t_after = s.timers()
        timers = {k: round((t_after[k] - t_before[k]) / args.steps, 4) for k in t_after}
        kind = "reference"
        sample = (f"{args.steps} GN matvecs of the compiled reference at {n}^3 (fp64, 1 thread; "
                  "the reference has no threading)")
    else:
        val, dt, kind, sample, timers = cpu_reference_sample(64, args.steps)
        n, same = 64, False
    value = n ** 3 * args.steps / dt / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"SYN {nx}x{ny}x{nz} GN Hessian matvec" +
                   ("" if same else f" (per-GPU {n}^3 sample on the host)"),
                   "grid": [nx, ny, nz], "nt": NT, "interp_degree": 3, "beta": BETA},
        "same_config_as_gpu_arm": same,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample,
                         "host_cores": os.cpu_count()},
        "reference_kernel_timers_s_per_matvec": timers,
        "fft_column": "FFTW3-API shim (oracle/shim/fftw_shim.c; FFTW3 is not installed)",
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# --------------------------------------------------------------- GPU leg ----

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2008_12820_b200.dist import init_from_env
    from paper_2008_12820_b200.solver import Config, Solver

    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE', '1')}")
    ctx, rank, world, local = init_from_env()

    dims = (args.size,) * 3 if world == 1 else weak_grid(args.size, world)
    if args.grid:  # explicit global grid (diagnostics), e.g. --grid 512,256,256
        dims = tuple(int(x) for x in args.grid.split(","))
    deg = args.degree
    Nvox = dims[0] * dims[1] * dims[2]

    # linearisation point through the solver C ABI, SYN inputs built on the
    # device (syn.cpp:9-49): v = 0.5 v_syn, vt = -g
    solver = Solver(ctx, dims, Config(continuation=False, beta_target=BETA, interp_degree=deg,
                                      nt=NT))
    solver.syn_images()
    g = solver.grid
    v = (0.5 * ctx.syn_velocity(g)).contiguous()
    solver.linearize(v, BETA)
    vt = (-solver.gradient()).contiguous()
    del v
    out = torch.empty_like(vt)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        solver.matvec(vt, out)

    for _ in range(max(args.warmup, 3 if args.warmup >= 3 else args.warmup)):
        step()
    barrier()

    # ---- timed region: K matvecs, inputs resident in HBM (> L2: no flush needed)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launches()
    ctx.enable_timers(True)
    t_before = ctx.timers()
    c_before = ctx.comm()
    with ClockSampler(local) as clk:
        barrier()
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launches() - l0
    ctx.enable_timers(False)
    kstats = ctx.kernel_stats()
    t_after = ctx.timers()
    c_after = ctx.comm()

    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = Nvox * args.steps / (ms * 1e-3) / 1e6
    # the timed matvec's result against the SURVEY §8c probe golden ||H vt||
    # (fp64 reference run, 256^3 SYN linearisation)
    hh = torch.tensor([float((out.double() ** 2).sum())], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(hh)
    h_norm = float(torch.sqrt(hh * (2 * math.pi) ** 3 / Nvox))
    golden = {(256, 256, 256): 9.8485730595e-2, (64, 64, 64): 9.8356971587e-2}.get(tuple(dims))
    check = {"H_norm": h_norm, "golden": golden,
             "rel": abs(h_norm / golden - 1) if golden and deg == 3 else None}

    # ---- e2e: the public API with HOST buffers, copies inside the timed region.
    # vreg_solver_matvec_host_async pipelines call k's upload, call k-1's
    # matvec and call k-2's download (PCIe is full duplex); every step's
    # H2D of its input and D2H of its result is inside the timed region,
    # which is host wall clock between full device synchronisations.
    h_in = [torch.empty(vt.shape, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    for h in h_in:
        h.copy_(vt)
    h_out = [torch.empty(vt.shape, dtype=torch.float32, pin_memory=True) for _ in range(2)]

    def run_e2e(k):
        for i in range(k):
            solver.matvec_host_async(h_in[i % 2], h_out[i % 2])
        solver.wait()

    run_e2e(2)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    run_e2e(args.steps)
    torch.cuda.synchronize()
    ms_e2e = (time.perf_counter() - t0) * 1e3
    barrier()
    # the pipelined result equals the blocking call's
    ref_out = torch.empty_like(h_out[0])
    solver.matvec_host(h_in[0], ref_out)
    e2e_diff = float((ref_out - h_out[(args.steps - 1) % 2]).norm() / ref_out.norm())
    t = torch.tensor([ms_e2e], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_e2e = float(t.item())
    e2e_value = Nvox * args.steps / (ms_e2e * 1e-3) / 1e6

    # ---- the other two BASELINE metrics (single GPU): 2LInvH0 preconditioner
    # apply throughput at this linearisation (configs[2]) and the full GNK
    # registration time with the reference defaults (configs[1]).
    extra = {}

    def max_over_ranks(x):
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if not args.no_registration:
        r = (-vt).contiguous()
        for _ in range(3):  # refresh + warm (coarse cuFFT plans, pool)
            solver.precond("2linvh0", r, 0.5)
        barrier()
        napp = 7
        inner = 0
        per = []
        for _ in range(napp):  # each apply bracketed by device syncs
            t0 = time.perf_counter()
            _, st = solver.precond("2linvh0", r, 0.5)
            torch.cuda.synchronize()
            per.append((time.perf_counter() - t0) * 1e3)
            inner += st["inner"]
        barrier()
        pms = max_over_ranks(sorted(per)[napp // 2])
        # where an apply's time goes (CUDA-event timers of the named scopes,
        # rank 0; outside the timed applies above)
        ctx.enable_timers(True)
        ctx.kernel_stats(reset=True)
        tb = ctx.timers()
        for _ in range(3):
            solver.precond("2linvh0", r, 0.5)
        torch.cuda.synchronize()
        ctx.enable_timers(False)
        ks, ta = ctx.kernel_stats(), ctx.timers()
        extra["precond_2linvh0"] = {"ms_per_apply": pms, "applies_per_s": 1e3 / pms,
                                    "ms_each": [round(x, 3) for x in per],
                                    "timing": "median of 7 host wall-clock applies, device-synced",
                                    "inner_cg_per_apply": inner / napp, "eps_k": 0.5,
                                    "timers_ms_per_apply": {
                                        k: round((ta[k] - tb[k]) / 3 * 1e3, 4)
                                        for k in ta if ta[k] != tb[k]},
                                    "scopes_ms_per_apply": {
                                        k: round(v["seconds"] / 3 * 1e3, 4) for k, v in ks.items()}}
        # twice: the first run pays cuFFT plan creation for the coarse grid
        # and the pool's first allocations; the second is the steady state
        secs = []
        for _ in range(2):
            reg = Solver(ctx, dims, Config(interp_degree=deg, nt=NT))  # optim.hpp:17-37 defaults
            reg.syn_images()
            barrier()
            t0 = time.perf_counter()
            _, rep, cnt = reg.register()
            torch.cuda.synchronize()
            barrier()
            secs.append(max_over_ranks(time.perf_counter() - t0))
            reg.close()
        extra["registration"] = {
            "seconds": secs[1], "seconds_first_run": secs[0],
            "grid": list(dims), "n_gpus": world, "config": "reference defaults: beta 1 -> 5e-4 "
            "continuation, 2LInvH0 (InvA above beta 0.5), eps_newton 5e-2, nt 4, cubic",
            "gn_iters": rep["total_gn"], "pcg_iters": rep["total_pcg"], "levels": rep["levels"],
            "mism_rel": rep["mism_rel"], "final_g_rel": rep["final_g_rel"],
            "phases_s": {k: rep[f"t_{k}"] for k in ("pc", "obj", "grad", "hess")}}
    # ---- trilinear matvec at the same linearisation (the paper's scaling runs
    # used linear interpolation; SURVEY §8d reports both)
    if deg == 3 and not args.no_linear:
        lin = Solver(ctx, dims, Config(continuation=False, beta_target=BETA, interp_degree=1,
                                       nt=NT))
        lin.syn_images()
        v1 = (0.5 * ctx.syn_velocity(g)).contiguous()
        lin.linearize(v1, BETA)
        vt1 = (-lin.gradient()).contiguous()
        del v1
        out1 = torch.empty_like(vt1)
        for _ in range(3):
            lin.matvec(vt1, out1)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            lin.matvec(vt1, out1)
        ev1.record(stream)
        barrier()
        lms = max_over_ranks(ev0.elapsed_time(ev1))
        extra["linear"] = {"interp_degree": 1, "value": Nvox * args.steps / (lms * 1e-3) / 1e6,
                           "unit": UNIT, "ms_per_step": lms / args.steps}
        lin.close()
        del vt1, out1
    nbytes = vt.numel() * 4

    if rank == 0:
        peak, peak_kind = measured_peak()
        # dominant kernel by device time inside the timed region
        dom = max(kstats.items(), key=lambda kv: kv[1]["seconds"]) if kstats else None
        roof = None
        BPV = {"sl_scatter_sweep": 28.0, "sl_inc_step": 24.0, "sl_assemble": 16.0 * (NT + 1) + 24.0,
               "sl_inc_init": 12.0 * (NT + 1) + 16 + 4.0 * NT, "spec_axis3": 24.0,
               "spec_axis2": 36.0, "spec_axis1": 36.0}
        # every timed kernel group of the matvec against the same peak (the
        # dominant one below is the headline `roofline`)
        by_kernel = {}
        for kname, kst in kstats.items():
            if kname in BPV and kst["count"]:
                per = kst["seconds"] / kst["count"]
                ach = BPV[kname] * (Nvox // world) / per / 1e9
                by_kernel[kname] = {"launch_us": round(per * 1e6, 1), "launches": kst["count"],
                                    "bytes_per_voxel": BPV[kname], "achieved_gbs": round(ach, 1),
                                    "frac": round(ach / peak, 3)}
        extra["roofline_by_kernel"] = by_kernel
        if dom:
            name, st = dom
            per_launch_s = st["seconds"] / max(st["count"], 1)
            Nloc = Nvox // world
            bpv = BPV.get(name)
            traffic = ncu_traffic()
            roof = {"bound": "hbm", "kernel": name, "peak": peak, "peak_kind": peak_kind,
                    "unit": "GB/s", "bytes_per_voxel": bpv,
                    "launch_us": per_launch_s * 1e6, "launches": st["count"],
                    "traffic": (traffic or {}).get(name)}
            if bpv:
                ach = bpv * Nloc / per_launch_s / 1e9
                roof.update({"achieved": ach, "frac": ach / peak})
            # the SL sweeps are shared-memory-pipe bound (64 taps / point):
            # wavefronts per launch vs one wavefront per SM clock
            wf = ncu_smem_wavefronts().get(name)
            sm_hz = (clk.summary().get("sm_mhz") or 0) * 1e6
            if wf and sm_hz:
                nsm = torch.cuda.get_device_properties(local).multi_processor_count
                roof["smem_pipe"] = {"wavefronts_per_launch": wf,
                                     "frac": wf / (per_launch_s * nsm * sm_hz),
                                     "peak": "1 wavefront / SM / clock"}
        matvec_bytes = bytes_per_voxel(NT) * (Nvox // world)
        share = {k: round(v["seconds"] / (ms * 1e-3) , 4) for k, v in kstats.items()}
        fft_s = t_after["fft"] - t_before["fft"]
        cpu = None
        if world == 1 and not args.no_cpu:
            val, dt, kind, sample, timers = cpu_reference_sample(dims[0] if dims[0] == dims[1] == dims[2] else 64, 1)
            cpu = {"value": val, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample,
                   "seconds": dt, "host_cores": os.cpu_count(),
                   "reference_kernel_timers_s": timers, "fft_column": "FFTW3-API shim"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"SYN {dims[0]}x{dims[1]}x{dims[2]} GN Hessian matvec",
                       "grid": list(dims), "nt": NT, "interp_degree": deg, "beta": BETA,
                       "precond": None, "parallelism": f"x1-slab x{world}",
                       "l2": "inputs > L2 (grads+chars+vt ~ %.1f GB/GPU)" % (
                           (3 * (NT + 1) + 6) * 4 * Nvox / world / 1e9)},
            "matvec_per_s": args.steps / (ms * 1e-3),
            "matvec_gbs": matvec_bytes / (ms / args.steps * 1e-3) / 1e9,
            "matvec_bytes_per_voxel": {"survey_fused_min": bytes_per_voxel(NT),
                                       "ours_moved": bytes_per_voxel_ours(NT)},
            "matvec_frac_of_hbm": matvec_bytes / (ms / args.steps * 1e-3) / 1e9 / peak,
            "fft_ms_per_step": fft_s / args.steps * 1e3,
            "nvlink": None if world == 1 else {
                # bytes each GPU sends per matvec (halos, reverse halos, regulariser
                # transposes) and the NVLink 5 time they would take alone
                "bytes_per_matvec": sum(c_after[k] - c_before[k] for k in (
                    "ghost_interp_bytes", "scatter_points_bytes", "fft_transpose_bytes",
                    "ghost_fd_bytes", "reduce_bytes")) / args.steps,
                "peak_gbs_per_direction": 900.0,
                "ms_at_peak": sum(c_after[k] - c_before[k] for k in (
                    "ghost_interp_bytes", "scatter_points_bytes", "fft_transpose_bytes",
                    "ghost_fd_bytes", "reduce_bytes")) / args.steps / 900e9 * 1e3,
                "comm_timer_ms": round(sum((t_after[k] - t_before[k]) for k in (
                    "interp_comm", "scatter_comm", "transpose_comm")) / args.steps * 1e3, 4),
                **nvlink_roofline(c_before, c_after, t_before, t_after, args.steps)},
            "timer_ms_per_step": {k: round((t_after[k] - t_before[k]) / args.steps * 1e3, 4)
                                  for k in t_after if t_after[k] != t_before[k]},
            "kernel_share": share,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes, "ms_per_step": ms_e2e / args.steps,
                    "api": "vreg_solver_matvec_host_async (pinned host buffers, 2 slots)",
                    "rel_diff_vs_blocking_call": e2e_diff},
            "result_check": check,
            "gpu_launches": launches,
            "sl_tiles": dict(zip(("built", "over_smem_budget"), ctx.tile_stats())),
            "clocks": clk.summary(),
            **extra,
        }
        emit(line)
    solver.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


NVLINK_PEER_GBS = 770.0   # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def nvlink_roofline(c0, c1, t0, t1, steps):
    """NVLink roofline of the exchanges: bytes each GPU sends per matvec over
    the time the comm timers saw them take (halos, reverse halos, regulariser
    transposes), against the measured 770 GB/s peer copy per direction."""
    keys_b = ("ghost_interp_bytes", "scatter_points_bytes", "fft_transpose_bytes",
              "ghost_fd_bytes", "reduce_bytes")
    keys_t = ("interp_comm", "scatter_comm", "transpose_comm")
    b = sum(c1[k] - c0[k] for k in keys_b) / steps
    t = sum(t1[k] - t0[k] for k in keys_t) / steps
    if t <= 0:
        return {}
    ach = b / t / 1e9
    return {"achieved_gbs": ach, "peak_gbs": NVLINK_PEER_GBS, "peak_kind": "measured peer copy",
            "frac": ach / NVLINK_PEER_GBS}


_JSON_FD = None


def emit(line: dict):
    """Write the ONE JSON result line to the real stdout (fd 1 is pointed at
    stderr while we run, so library banners -- e.g. NCCL's version line --
    cannot interleave with it)."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=256, help="per-GPU cube edge (weak scaling family)")
    ap.add_argument("--degree", type=int, default=3)
    ap.add_argument("--no-linear", action="store_true", help="skip the trilinear matvec line")
    ap.add_argument("--grid", default="", help="explicit global grid n1,n2,n3 (overrides --size)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-registration", action="store_true",
                    help="skip the registration-time and preconditioner extras")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
