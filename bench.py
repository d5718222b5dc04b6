#!/usr/bin/env python
"""Benchmark: the recycled-Krylov global-basis build on B200 (BASELINE.json
metric: recycled-Krylov solves/s and basis-build time at 3D 128^3).

Workload: config C4 (3D 128^3, n = 2,097,152, complex128, 96 RHS, k = 64,
16 systems = 8 parameter points x omega/nu in {0, 0.1}, candidate cap 768,
RRQR at 1e-10), the configuration the metric is quoted on.

* One *step* = one ``process_system`` (proj/src/basis.cpp:157-207) of the
  build, in build order: timed step i is system (i mod 16) + 1 of build
  floor(i / 16). A build starts from the (offline, paper section 5.3) seed
  U0 / X0 on a fresh basis and its 16th step ends with the Algorithm-1 RRQR
  compression of the candidate basis. No system is ever revisited on a basis
  that already holds it. Warm-up steps run on a throw-away basis.
* ``value`` = (system, RHS) solves with >= 1 inner iteration / device time of
  the K timed steps (CUDA events on the library stream), inputs (coefficient
  fields, seed) resident in HBM, solutions written to device memory.
* ``basis_build_s`` = the device time of one complete build: seed (device
  Lanczos U0 + batched CG/COCG X0) + systems 1..16 + RRQR (the systems of
  build 0 that the timed window does not cover are run after it).
* ``e2e`` = the same K steps through the public Python API
  (``romdot.process_system``) with HOST inputs: per step the fields are
  copied H2D from pinned memory and the n x 96 solution block D2H inside the
  timed region (wall clock around the region, after a device sync).
* ``roofline`` = the dominant kernel (``cg_fused``, the one-solve iteration of
  the systems before the candidate cap): algorithmic bytes n (es (c + 10) + 32)
  per launch over its live CUDA-event-timed launch duration, peak =
  MEASURED_PEAKS.json hbm_gbs. ``roofline.batched`` is the same for one step of
  the batched iteration that runs the independent right-hand sides after the
  cap (16 solves in flight, bcg_defl.cuh). ``fp64`` adds the DMMA Gram / tall
  GEMM rates against a cuBLAS DGEMM peak measured in the same run.
* ``cpu_baseline`` = the CPU checker (the reference's own sources compile into
  oracle/_ref, but they are 2D / real / MINRES only and cannot run C4) timed
  on the box's host cores on ONE complete C4 (system, RHS) step
  -- global check, recycle space from_raw, recycled COCG to 0.25 tol, X_j,
  append decision -- replayed from the device's state during warm-up
  (oracle/replay.py).
* ``--impl reference``: the same checker on 4 complete C4 (system, RHS) steps
  spread over the build (pre- and post-cap, omega = 0 and 0.1), replayed from
  the device's state; the device build that produces those states is untimed
  setup, the timed region is CPU only.

Multi-GPU: the basis build is causally sequential -- N GPUs
run N independent replicas ("replicas only"); value = all ranks' solves / max
rank device time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1602_00138_b200 import problem as P  # noqa: E402

METRIC = "recycled-Krylov solves/s (3D 128^3 basis build)"
UNIT = "solves/s"


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        pw = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows),
                "power_w_median": statistics.median(pw) if pw else None}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def aggregate_replicas(dist, device, solves, t_ms, e2e_ms=None):
    """Replicas only: whole-job solves = sum over ranks, time =
    max over ranks (device-timed). Returns (solves_all, t_max_ms, e2e_max_ms)."""
    import torch
    t = torch.tensor([float(t_ms)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = torch.tensor([float(solves)], device=device, dtype=torch.float64)
    dist.all_reduce(s)
    te = None
    if e2e_ms is not None:
        e = torch.tensor([float(e2e_ms)], device=device, dtype=torch.float64)
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
        te = float(e.item())
    return int(round(s.item())), float(t.item()), te


# ------------------------------------------------------------ device build ---
class Build:
    """One config on the device through the public API (romdot.py): fields of
    every system (pinned host + device copies), the device seed, fresh bases,
    process_system steps and the RRQR compression, device-timed."""

    def __init__(self, cfg: P.ProblemConfig, ctx, local: int):
        import torch
        from paper_1602_00138_b200 import romdot as R
        self.R, self.torch, self.cfg, self.ctx, self.local = R, torch, cfg, ctx, local
        self.g, self.lay = cfg.grid, cfg.layout()
        self.n, self.nrhs = self.g.n, self.lay.n_rhs
        self.dt = np.dtype(cfg.dtype)
        self.tdt = torch.complex128 if cfg.complex else torch.float64
        self.systems = cfg.systems()
        t0 = time.perf_counter()
        self.pin, self.dev = [], []
        for pt, w in self.systems:
            f = cfg.fields(pt, w)
            hD = torch.from_numpy(f.D).pin_memory()
            hm = torch.from_numpy(f.mu).pin_memory()
            self.pin.append(P.Fields(hD.numpy(), hm.numpy(), f.shift))
            self.dev.append((hD.cuda(local), hm.cuda(local), f.shift))
        self.f0 = cfg.fields(0)
        torch.cuda.synchronize()
        self.field_gen_s = time.perf_counter() - t0
        self.op = R.SchurOperator(self.g, self.f0, self.dt, ctx)
        self.X = torch.empty((self.nrhs, self.n), dtype=self.tdt, device=f"cuda:{local}")

    def timed(self, fn):
        self.ctx.mark()
        out = fn()
        self.ctx.mark()
        return out, self.ctx.elapsed_ms()

    def seed(self):
        """init_basis (basis.cpp:136-155): U0 by device shift-invert Lanczos, X0
        by batched device CG/COCG at 0.25 tol. Returns device seconds."""
        R, torch, cfg = self.R, self.torch, self.cfg
        op_r = R.SchurOperator(self.g, self.f0, np.float64, self.ctx)
        U0 = torch.empty((cfg.k, self.n), dtype=torch.float64, device=f"cuda:{self.local}")
        lam = np.zeros(cfg.k)
        L = R.load_library()

        def eig():
            R._check(L.rd_smallest_eigenpairs(op_r.h, cfg.k, min(cfg.tol, 1e-8), R._p(lam), U0.data_ptr(),
                                              R.DEVICE))
        _, t_eig = self.timed(eig)
        self.X0 = torch.empty((self.nrhs, self.n), dtype=self.tdt, device=f"cuda:{self.local}")
        idx = np.ascontiguousarray(self.lay.idx, dtype=np.int64)
        val = np.ascontiguousarray(self.lay.val, dtype=np.float64)
        tot = C.c_long()

        def x0():
            R._check(L.rd_initial_solutions(self.op.h, R._dt(self.dt), self.nrhs, R._p(idx), R._p(val), cfg.tol,
                                            self.X0.data_ptr(), R.DEVICE, C.byref(tot)))
        _, t_x0 = self.timed(x0)
        self.U0 = U0.to(self.tdt) if cfg.complex else U0
        self.lam = lam
        self.seed_info = {"eigenpairs_U0_s": t_eig / 1e3, "X0_solves_s": t_x0 / 1e3, "X0_iterations": tot.value,
                          "lambda_min": float(lam[0])}
        return (t_eig + t_x0) / 1e3

    def new_basis(self):
        return self.R.GlobalBasis.from_device(self.U0.data_ptr(), self.X0.data_ptr(), self.n, self.cfg.k,
                                              self.nrhs, self.dt, self.cfg.cap, self.ctx)

    def step(self, gb, s: int, host: bool = False, Xhost=None):
        """System s (0-based) of the build: fields from device memory, X on the
        device -- or, host=True, fields from pinned host memory and X to Xhost."""
        R = self.R
        if host:
            self.op.set_fields(self.pin[s], where=R.HOST)
            return R.process_system(gb, self.op, self.lay, self.cfg.tol, s + 1, X_out=Xhost)
        D, mu, sh = self.dev[s]
        self.op.set_fields(P.Fields(None, None, sh), where=R.DEVICE, D_ptr=D.data_ptr(), mu_ptr=mu.data_ptr())
        return R.process_system(gb, self.op, self.lay, self.cfg.tol, s + 1, X_out=self.X.data_ptr())

    def residual_max(self) -> float:
        res = self.R.residual_norms(self.op, self.lay, self.X.data_ptr(), self.R.DEVICE)
        return float(res.max())


def solves_of(pr) -> int:
    return sum(1 for r in pr.log if r.iterations > 0)


def full_build(cfg, ctx, local) -> dict:
    """Seed + all systems + RRQR of a config, device-timed (the BASELINE.md
    table's GPU column for C1-C3)."""
    b = Build(cfg, ctx, local)
    t_seed = b.seed()
    gb = b.new_basis()
    t_sys = 0.0
    solves = its = 0
    worst = 0.0
    for s in range(len(b.systems)):
        pr, ms = b.timed(lambda: b.step(gb, s))
        t_sys += ms / 1e3
        solves += solves_of(pr)
        its += pr.inner_iterations
        worst = max(worst, b.residual_max())
    (rank, _, _), ms = b.timed(lambda: gb.compress(1e-10))
    gb.destroy()
    return {"basis_build_s": round(t_seed + t_sys + ms / 1e3, 3), "seed_s": round(t_seed, 3),
            "systems_s": round(t_sys, 3), "rrqr_s": round(ms / 1e3, 3), "solves": solves, "inner_iterations": its,
            "solves_per_s": round(solves / t_sys, 2), "rank": int(rank), "n": b.n, "rhs": b.nrhs,
            "systems": len(b.systems), "max_explicit_residual": worst, "tol": cfg.tol}


def fp64_rates(ctx, n: int) -> dict:
    """FP64 tensor-pipe evidence: cuBLAS DGEMM (torch.matmul, 8192^3) as the
    measured FP64 peak, against this library's DMMA Gram (V^H V at the refresh
    width, complex) and tall GEMM on the same box."""
    import torch
    from paper_1602_00138_b200 import romdot as R
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    peak = 2 * 8192 ** 3 / (best / 1e3) / 1e12
    del a, b
    torch.cuda.empty_cache()
    out = {"peak_tflops": round(peak, 2), "peak_kind": "measured: cuBLAS DGEMM 8192^3 (torch.matmul fp64), best of 5"}
    for name, (m, cplx) in {"gram_c128_r768": (768, True), "gram_f64_r594": (594, False)}.items():
        ms = R.bench_gram(n, m, m, cplx, True, iters=3, ctx=ctx)
        fl = (8.0 if cplx else 2.0) * n * m * m / 2.0  # SYRK flops (half of the GEMM)
        ach = fl / (ms / 1e3) / 1e12
        out[name] = {"ms": round(ms, 3), "tflops": round(ach, 2), "frac": round(ach / peak, 3),
                     "flops": "SYRK: (8 complex | 2 real) n m^2 / 2"}
    ms = R.bench_gemm(n, 768, 768, True, upper=False, iters=3, ctx=ctx)
    fl = 8.0 * n * 768 * 768
    out["gemm_tall_c128_768"] = {"ms": round(ms, 3), "tflops": round(fl / (ms / 1e3) / 1e12, 2),
                                 "frac": round(fl / (ms / 1e3) / 1e12 / peak, 3), "flops": "8 n m k (complex)"}
    return out


# ------------------------------------------------------------------ main ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1-C3 full builds")
    ap.add_argument("--no-fp64", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = P.CONFIGS[args.config]

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank, local)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)

    from paper_1602_00138_b200 import build, romdot as R
    build.build()
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    ctx = R.Context(local)
    b = Build(cfg, ctx, local)
    ns = len(b.systems)
    t_seed = b.seed()
    log(f"seed: {t_seed:.2f}s {b.seed_info}")

    def barrier():
        torch.cuda.synchronize()
        ctx.sync()
        if dist is not None:
            dist.barrier()

    # ---- warm-up on a throw-away basis (+ the CPU baseline sample) ---------
    gb = b.new_basis()
    cpu = None
    smp = None
    want_cpu = rank == 0 and world == 1 and not args.no_cpu
    if want_cpu:
        import replay as RP
        import oracle as orc
        cpu_pt = {2: [b.lay.n_src + 17]}  # a detector RHS of system 2 (omega/nu = 0.1, COCG)
        smp = RP.Sampler(gb, cfg, b.lay, cpu_pt, cfg.cap, cfg.tol, verbose=False)
        gb.set_rhs_hook(smp)
    warm_ms = []
    for i in range(args.warmup):
        s = i % ns
        if smp is not None:
            pt, w = b.systems[s]
            smp.set_operator(orc.Operator.grid(b.g, b.pin[s], b.dt))
        pr, ms = b.timed(lambda: b.step(gb, s))
        if smp is not None:
            smp.compare_system(s + 1, pr.log, None)
        warm_ms.append(round(ms, 1))
        log(f"warmup system {s + 1}: {ms:.0f} ms, {pr.inner_iterations} its, {pr.appends} appends")
    if smp is not None:
        gb.set_rhs_hook(None)
        cps = [cp for cp in smp.results if cp.device_row is not None]
        if cps:
            cp = cps[0]
            t = cp.replay.times["total"]
            cpu = {"value": (1.0 if cp.replay.iterations > 0 else 0.0) / t, "unit": UNIT, "cores": host_cores(),
                   "kind": "port",
                   "sample": f"one complete C4 (system {cp.system}, RHS {cp.rhs}) step on the CPU checker "
                             f"(oracle/romdot_oracle.cpp replay_rhs) from the device state: global check over "
                             f"K_img ({cp.cols} cols), from_raw of U_j ({len(cp.space)} cols), recycled COCG to "
                             f"0.25 tol ({cp.replay.iterations} its; device {cp.device_row[1]}), X_j, append "
                             f"decision; {host_cores()} OpenMP threads",
                   "phase_s": {k: round(v, 3) for k, v in cp.replay.times.items()}}
        del smp
    gb.destroy()
    del gb

    # ---- timed: K steps of the build, device-resident inputs ---------------
    # per-step device times from events on the library stream (no extra syncs)
    lib_stream = torch.cuda.ExternalStream(ctx.stream)

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(lib_stream)
        return e

    launches0 = ctx.launches
    ctx.profile(True)
    solves = its_tot = zeros = 0
    per_step = []
    marks = []          # (step, start event, rrqr event or None)
    b0 = {"solves": 0, "its": 0, "rank": None}
    gb = None
    barrier()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" selects the timed launches
    with ClockSampler(local) as clk:
        ctx.mark()
        for i in range(args.steps):
            s = i % ns
            e_start = ev()
            if s == 0:
                if gb is not None:
                    gb.destroy()
                gb = b.new_basis()
            pr = b.step(gb, s)
            e_rr = None
            ns_ = solves_of(pr)
            solves += ns_
            zeros += sum(1 for r in pr.log if r.iterations == 0)
            its_tot += pr.inner_iterations
            if i < ns:
                b0["solves"] += ns_
                b0["its"] += pr.inner_iterations
            if s == ns - 1:
                e_rr = ev()
                rk, _, _ = gb.compress(1e-10)
                if i // ns == 0:
                    b0["rank"] = int(rk)
            marks.append((i, e_start, e_rr))
            per_step.append([i // ns, s + 1, pr.inner_iterations, pr.appends, gb.cols])
        e_end = ev()
        ctx.mark()
        barrier()
    torch.cuda.nvtx.range_pop()
    t_val_ms = ctx.elapsed_ms()
    launches = ctx.launches - launches0
    prof = ctx.prof()
    ctx.profile(False)
    worst = b.residual_max()  # the last timed system's 96 solutions (X still on the device)
    for row in per_step:
        log(f"timed build {row[0]} system {row[1]}: {row[2]} its, {row[3]} appends, cols={row[4]}")
    step_ms = []
    rr_ms = None
    for k, (i, e0, err) in enumerate(marks):
        e1 = marks[k + 1][1] if k + 1 < len(marks) else e_end
        step_ms.append(e0.elapsed_time(e1))
        if err is not None and i // ns == 0:
            rr_ms = err.elapsed_time(e1)

    # ---- one complete build's device time (seed + 16 systems + RRQR) -------
    # build 0 = the first 16 timed steps; systems the window did not reach run
    # now on the same basis (device events), then its RRQR
    sys_ms = [round(x, 1) for x in step_ms[:ns]]
    if rr_ms is not None:
        sys_ms[ns - 1] = round(step_ms[ns - 1] - rr_ms, 1)
    else:
        if args.steps < ns:
            for s in range(args.steps, ns):
                pr, ms = b.timed(lambda: b.step(gb, s))
                sys_ms.append(round(ms, 1))
                b0["solves"] += solves_of(pr)
                b0["its"] += pr.inner_iterations
        (rk, _, _), rr_ms = b.timed(lambda: gb.compress(1e-10))
        b0["rank"] = int(rk)
    build_s = t_seed + sum(sys_ms) / 1e3 + rr_ms / 1e3
    if gb is not None:
        gb.destroy()
        gb = None

    # ---- e2e: the same K steps through the public API with host buffers ---
    e2e = None
    if not args.no_e2e:
        Xhost = torch.empty((b.nrhs, b.n), dtype=b.tdt).pin_memory().numpy().T  # Fortran (n, nrhs) view
        s2 = 0
        barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            s = i % ns
            if s == 0:
                if gb is not None:
                    gb.destroy()
                gb = b.new_basis()
            pr = b.step(gb, s, host=True, Xhost=Xhost)
            s2 += solves_of(pr)
            if s == ns - 1:
                gb.compress(1e-10)
        barrier()
        t_e2e_ms = (time.perf_counter() - t0) * 1e3
        if gb is not None:
            gb.destroy()
            gb = None
        e2e = {"value": s2 / (t_e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * b.n * 8,
               "d2h_bytes_per_step": b.n * b.nrhs * b.dt.itemsize + b.nrhs * 5 * 8, "ms": t_e2e_ms,
               "api": "romdot.process_system(..., X_out=pinned host array) + SchurOperator.set_fields(host)"}

    # ---- multi-rank aggregation (replicas) ---------------------------------
    t_max, solves_all = t_val_ms, solves
    if dist is not None:
        solves_all, t_max, te = aggregate_replicas(dist, f"cuda:{local}", solves, t_val_ms,
                                                   e2e["ms"] if e2e is not None else None)
        if e2e is not None:
            e2e["value"] = solves_all / (te / 1e3)
    value = solves_all / (t_max / 1e3) if t_max > 0 else 0.0

    # ---- roofline from the live samples ------------------------------------
    peak, peak_kind = measured_peaks()
    classes = {}
    for name, (ms, by, nsmp) in prof.items():
        if nsmp and name != "bcg_defl_slot_steps":
            classes[name] = {"ms_per_launch": ms / nsmp, "GBps": by / (ms / 1e3) / 1e9, "samples": nsmp,
                             "bytes_per_launch": by / nsmp}
    roofline = None
    if classes:
        dom = max(classes, key=lambda k: prof[k][0])
        ach = classes[dom]["GBps"]
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak, "peak_kind": peak_kind,
                    "unit": "GB/s", "frac": round(ach / peak, 4), "per_class": classes,
                    "algorithmic_bytes": "n (es (c + 10) + 32) per launch: K (n x c, es = 16 B) read once, "
                                         "r, w, p, s, y (+ x-tile reuse) and the 4 coefficient planes"}
        try:
            ref = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))  # committed ncu summary
            k = ref["kernels"][dom]
            ratio = (k["dram_read_bytes"] + k["dram_write_bytes"]) / k["algorithmic_bytes"]
            roofline.update({"traffic": round(classes[dom]["bytes_per_launch"] * ratio),
                             "traffic_unit": "bytes per launch (DRAM read + write)",
                             "traffic_over_algorithmic": round(ratio, 4), "traffic_source": k["source"]})
        except Exception:
            roofline["traffic"] = None
        # device-time share of the dominant class: cg_fused runs once per inner iteration of
        # the one-solve path; the batched steps are all sampled (time = their sum)
        batched_ms = prof.get("bcg_defl_step", (0.0, 0.0, 0))[0]
        batched_its = prof.get("bcg_defl_slot_steps", (0.0, 0.0, 0))[2]
        if dom == "cg_fused" and t_val_ms:
            roofline["share_of_step"] = round(classes[dom]["ms_per_launch"] * (its_tot - batched_its) / t_val_ms, 3)
        elif dom == "bcg_defl_step" and t_val_ms:
            roofline["share_of_step"] = round(batched_ms / t_val_ms, 3)
        else:
            roofline["share_of_step"] = None
        if "bcg_defl_step" in classes:
            bc = classes["bcg_defl_step"]
            roofline["batched"] = {
                "kernel": "bcg_defl step (stencil_tma, bd_dots, bd_T_eig, bd_T_trail, bd_coef, bd_N_eig, bd_update)",
                "achieved": round(bc["GBps"], 1), "frac": round(bc["GBps"] / peak, 4), "steps": bc["samples"],
                "ms_per_step": round(bc["ms_per_launch"], 4), "share_of_step": round(batched_ms / t_val_ms, 3),
                "solve_iterations": batched_its,
                "algorithmic_bytes": "per step es n 2k (eigen block, T and N pass) + 32 n (coefficient planes); per "
                                     "slot-step es n (2 t + 15): trailing block twice and 15 vector passes",
            }

    fp64 = None
    if not args.no_fp64:
        try:
            fp64 = fp64_rates(ctx, b.n)
        except Exception as e:
            fp64 = {"error": str(e)}

    configs = {}
    if not args.no_configs and rank == 0:
        for name in ("C1", "C2", "C3"):
            try:
                configs[name] = full_build(P.CONFIGS[name], ctx, local)
                log(f"{name}: {configs[name]}")
            except Exception as e:
                configs[name] = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "c128" if cfg.complex else "f64", "data": "synthetic (seeded Gaussian-RBF level sets)",
            "config": {"workload": f"{cfg.name}: {b.g.d}D {b.g.N[0]}^{b.g.d} (n={b.n}), {b.nrhs} RHS, k={cfg.k}, "
                                   f"omega/nu in {list(cfg.omegas)}, tol={cfg.tol}, cap={cfg.cap}, RRQR 1e-10",
                       "step": "one process_system of the build in order (system = step mod 16 + 1; a new build "
                               "from the offline seed every 16 steps, RRQR at its end)",
                       "l2": "inputs larger than L2 (basis n x r streamed every iteration)",
                       "parallelism": f"replicas x{world}"},
            "solves": solves, "zero_iteration_rhs": zeros, "inner_iterations": its_tot,
            "iterations_per_solve": round(its_tot / max(1, solves), 2),
            "iterations_per_s": its_tot / (t_val_ms / 1e3) if t_val_ms else 0.0,
            "basis_build_s": round(build_s, 3), "basis_build_without_seed_s": round(build_s - t_seed, 3),
            "build": {"seed_s": round(t_seed, 3), **b.seed_info, "systems_ms": sys_ms, "rrqr_ms": round(rr_ms, 1),
                      "rank": b0["rank"], "candidate_cols": cfg.cap, "solves": b0["solves"],
                      "inner_iterations": b0["its"],
                      "max_explicit_residual_last_system": worst, "residual_ok": worst <= cfg.tol},
            "warmup_system_ms": warm_ms, "steps_detail": per_step,
            "step_ms": [round(x, 1) for x in step_ms],
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "fp64": fp64,
            "cpu_baseline": cpu, "configs": configs,
            "clocks": clk.summary(), "field_gen_s": round(b.field_gen_s, 2),
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


# ------------------------------------------------------------- reference ---
def run_reference(args, cfg, world, rank, local):
    """--impl reference: the CPU checker (restatement of the reference's CPU
    path; the reference's own sources compile into oracle/_ref but are 2D, real
    and MINRES only, so they cannot run the 3D complex C4 workload) on the box's
    host cores. The timed region is m = 4 complete C4 (system, RHS) steps on
    the CPU (global check over K_img, from_raw of U_j, recycled COCG to 0.25
    tol, X_j = correction + solve_projected, append decision), replayed from
    the basis state a device build reaches at those points (untimed setup).
    value = iterating solves / CPU seconds of those steps; the K reported
    steps share that fixed sample (ms_per_step = total / K). Warm-up: W
    zero-iteration replays (global check + solve_projected) at the first
    point. Also: one full C1 build on the checker (measured, single config)."""
    if rank != 0:
        return
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    cores = host_cores()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    import oracle as orc
    import replay as RP
    from paper_1602_00138_b200 import build, romdot as R
    build.build()
    torch.cuda.set_device(local)
    ctx = R.Context(local)
    b = Build(cfg, ctx, local)
    ns = len(b.systems)
    b.seed()
    nsrc = b.lay.n_src
    # pre-cap omega/nu = 0.1 (system 2) and 0 (7); post-cap 0.1 (12) and 0 (15)
    pts = {2: [nsrc + 17], 7: [4], 12: [nsrc + 41], 15: [12]}
    last = max(pts)
    gb = b.new_basis()
    smp = RP.Sampler(gb, cfg, b.lay, pts, cfg.cap, cfg.tol, keep_x=False, verbose=True)
    warm = {"done": False, "s": []}

    def hook(system, j):
        if not warm["done"] and j in smp.points.get(system, ()):
            V = gb.get_into(0, smp.Vb)
            K = gb.get_into(1, smp.Kb)
            Rm = gb.R
            for _ in range(args.warmup):  # zero-iteration path (tol = 1): global check + solve_projected
                rr = orc.replay_rhs(smp.op_o, V, K, Rm, gb.space(j), int(b.lay.idx[j]), float(b.lay.val[j]), 1.0,
                                    cfg.cap)
                warm["s"].append(round(rr.times["total"], 3))
            warm["done"] = True
        smp(system, j)

    gb.set_rhs_hook(hook)
    for s in range(last):
        pt, w = b.systems[s]
        smp.set_operator(orc.Operator.grid(b.g, b.pin[s], b.dt))
        if (s + 1) not in pts:
            smp.points.pop(s + 1, None)
        pr = b.step(gb, s)
        smp.compare_system(s + 1, pr.log, None)
        log(f"reference setup: device system {s + 1} done, cols={gb.cols}")
    gb.set_rhs_hook(None)
    gb.destroy()
    cps = smp.results
    t_cpu = sum(cp.replay.times["total"] for cp in cps)
    nsolve = sum(1 for cp in cps if cp.replay.iterations > 0)
    v = nsolve / t_cpu
    # C1 (2D 129^2, real): one whole build on the checker, seed included
    c1 = P.CONFIGS["C1"]
    t0 = time.perf_counter()
    g1, lay1 = c1.grid, c1.layout()
    f10 = c1.fields(0)
    _, U01 = orc.smallest_eigenpairs(orc.Operator.grid(g1, f10), c1.k, min(c1.tol, 1e-8))
    X01, _ = orc.initial_solutions(orc.Operator.grid(g1, f10, c1.dtype), lay1, c1.tol)
    gbo = orc.GlobalBasis(U01.astype(c1.dtype), X01, c1.cap)
    s1 = i1 = 0
    for si, (pt, w) in enumerate(c1.systems(), start=1):
        po = orc.process_system(gbo, orc.Operator.grid(g1, c1.fields(pt, w), c1.dtype), lay1, c1.tol, si)
        s1 += sum(1 for r in po.log if r.iterations > 0)
        i1 += po.inner_iterations
    rk1, _, _, _ = orc.qrcp(gbo.V, 1e-10, True)
    c1_s = time.perf_counter() - t0
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_cpu * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128" if cfg.complex else "f64", "data": "synthetic (seeded Gaussian-RBF level sets)",
            "config": {"workload": f"{cfg.name}: {b.g.d}D {b.g.N[0]}^{b.g.d} (n={b.n}), {b.nrhs} RHS, k={cfg.k}, "
                                   f"omega/nu in {list(cfg.omegas)}, tol={cfg.tol}, cap={cfg.cap}, RRQR 1e-10",
                       "step": "one process_system of the build in order (system = step mod 16 + 1; a new build "
                               "from the offline seed every 16 steps, RRQR at its end)",
                       "l2": "inputs larger than L2 (basis n x r streamed every iteration)",
                       "parallelism": f"replicas x{world}"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{len(cps)} complete C4 (system, RHS) steps on the CPU checker, replayed "
                                       f"from the device build's state at {[[cp.system, cp.rhs] for cp in cps]} "
                                       f"(global check, from_raw, recycled COCG to 0.25 tol, X_j, append decision); "
                                       f"K steps share this sample; per-system refresh not included (favours "
                                       f"the CPU)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_seconds": round(t_cpu, 2), "solves": nsolve,
            "inner_iterations": sum(cp.replay.iterations for cp in cps),
            "points": [{"system": cp.system, "rhs": cp.rhs, "cols": cp.cols, "cj": len(cp.space),
                        "its_cpu": cp.replay.iterations, "its_gpu": cp.device_row[1] if cp.device_row else None,
                        "appended_cpu": cp.replay.appended,
                        "appended_gpu": cp.device_row[2] if cp.device_row else None,
                        "phase_s": {k: round(x, 3) for k, x in cp.replay.times.items()}} for cp in cps],
            "warmup_s": warm["s"],
            "configs": {"C1": {"cpu_build_s": round(c1_s, 2), "solves": s1, "inner_iterations": i1,
                               "rank": int(rk1), "cores": cores, "note": "checker seed + 4 systems + QRCP"}},
            "setup": "device build to system %d (untimed; produces the states replayed on the CPU)" % last}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
