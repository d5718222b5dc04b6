#!/usr/bin/env python
"""Benchmark: recycled-Krylov global-basis build on B200 (BASELINE.json metric).

One *step* = one ``process_system`` call: every right-hand side of one
(parameter point, omega) system of the workload config is checked against the
global basis and, if needed, solved by recycled CG/COCG with the per-RHS
recycle space, and new directions are appended (basis.cpp:157-207).

Metric: recycled-Krylov solves/s = (system, RHS) solves with >= 1 inner
iteration per second of device time over the K timed steps.

* ``value``: inputs (coefficient fields) already resident in HBM, solutions
  kept on the device (the C ABI with device pointers).
* ``e2e``: the same K steps re-run through the C ABI with HOST buffers from
  pinned memory -- per step the fields are copied H2D and the n x n_rhs
  solution block D2H inside the timed region. Both runs start from the same
  device-computed seed (U0 via device Lanczos, X0 via device CG); the build is
  bitwise deterministic so both runs execute identical arithmetic.
* ``roofline``: live CUDA-event samples of the dominant inner-iteration kernel
  class (the tall-skinny recycle-space projections) with their algorithmic
  bytes; peak = MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline``: the CPU oracle (a restatement of the reference, which
  cannot be built here) on a bounded sample of the same workload.

Multi-GPU: the basis build is causally sequential -- N GPUs
run N independent replicas ("replicas only"); value = all ranks' solves / max
rank time.
"""
from __future__ import annotations

import argparse
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
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------- workload ---
def workload_systems(cfg: P.ProblemConfig, count: int):
    sys_list = cfg.systems()
    out = []
    for i in range(count):
        out.append(sys_list[i % len(sys_list)])
    return out


def cpu_sample(cfg: P.ProblemConfig, width: int, mean_its: float, iters: int = 6, threads: int = 0):
    """Oracle on a bounded sample of the same workload: one recycle space of the
    GPU run's mean width (from_raw) plus `iters` inner COCG/CG iterations on the
    workload operator; extrapolated to solves/s with the GPU run's mean
    iterations per solve (global-basis check/append costs excluded)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    if threads:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    g, lay = cfg.grid, cfg.layout()
    pt, w = cfg.systems()[0]
    f = cfg.fields(pt, w)
    op = orc.Operator.grid(g, f, cfg.dtype)
    rng = np.random.default_rng(7)
    W = rng.standard_normal((g.n, width)).astype(cfg.dtype)
    t0 = time.perf_counter()
    AW = op.apply(W)
    rs = orc.RecycleSpace(W, AW)
    t_raw = time.perf_counter() - t0
    b = lay.dense(g.n, cfg.dtype)[:, 0] if g.n * lay.n_rhs < 5e8 else None
    if b is None:
        b = np.zeros(g.n, dtype=cfg.dtype)
        b[lay.idx[0]] = lay.val[0]
    t1 = time.perf_counter()
    res = orc.recycled_cg(op, rs, b, 1e-30, iters, abs(lay.val[0]))
    t_it = (time.perf_counter() - t1) / max(1, res.report.iterations)
    per_solve = t_raw + mean_its * t_it
    return {"value": 1.0 / per_solve, "t_from_raw_s": t_raw, "t_iter_s": t_it,
            "sample": f"oracle from_raw(c={width}) + {res.report.iterations} inner iterations on {cfg.name} "
                      f"(n={g.n}, {np.dtype(cfg.dtype).name}); extrapolated with {mean_its:.1f} its/solve; "
                      "global check/append excluded"}


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


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ main ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=6)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = P.CONFIGS[args.config]

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)

    from paper_1602_00138_b200 import build, romdot as R
    build.build()
    ctx = R.Context(local)
    g, lay = cfg.grid, cfg.layout()
    n, nrhs = g.n, lay.n_rhs
    dt = np.dtype(cfg.dtype)
    tdt = torch.complex128 if cfg.complex else torch.float64
    es = dt.itemsize
    systems = workload_systems(cfg, args.warmup + args.steps)

    # host fields for every step (generated once, pinned) + device copies
    t_gen = time.perf_counter()
    f0 = cfg.fields(0)
    step_fields = [cfg.fields(pt, w) for (pt, w) in systems]
    pin = []
    dev = []
    for f in step_fields:
        hD = torch.from_numpy(f.D).pin_memory()
        hm = torch.from_numpy(f.mu).pin_memory()
        pin.append((hD, hm, f.shift))
        dev.append((hD.cuda(local), hm.cuda(local), f.shift))
    t_gen = time.perf_counter() - t_gen
    torch.cuda.synchronize()

    def set_dev(op, i):
        D, mu, sh = dev[i]
        op.set_fields(P.Fields(None, None, sh), where=R.DEVICE, D_ptr=D.data_ptr(), mu_ptr=mu.data_ptr())

    # ---- seed: U0 (device shift-invert Lanczos), X0 (device CG/COCG) ------
    op = R.SchurOperator(g, f0, dt, ctx)
    op_r = R.SchurOperator(g, f0, np.float64, ctx)
    U0 = torch.empty((cfg.k, n), dtype=torch.float64, device=f"cuda:{local}")
    lam = np.zeros(cfg.k)
    ctx.sync()
    t0 = time.perf_counter()
    R._check(R.load_library().rd_smallest_eigenpairs(op_r.h, cfg.k, min(cfg.tol, 1e-8), R._p(lam),
                                                      U0.data_ptr(), R.DEVICE))
    t_eig = time.perf_counter() - t0
    log(f"U0: {cfg.k} eigenpairs in {t_eig:.2f}s, lambda[0..2]={lam[:3]}")
    X0 = torch.empty((nrhs, n), dtype=tdt, device=f"cuda:{local}")
    idx = np.ascontiguousarray(lay.idx, dtype=np.int64)
    val = np.ascontiguousarray(lay.val, dtype=np.float64)
    import ctypes as C
    tot = C.c_long()
    t0 = time.perf_counter()
    R._check(R.load_library().rd_initial_solutions(op.h, R._dt(dt), nrhs, R._p(idx), R._p(val), cfg.tol,
                                                   X0.data_ptr(), R.DEVICE, C.byref(tot)))
    t_x0 = time.perf_counter() - t0
    log(f"X0: {nrhs} solves, {tot.value} iterations in {t_x0:.2f}s")
    U0c = U0.to(tdt) if cfg.complex else U0
    del U0

    def new_basis():
        h = C.c_void_p()
        R._check(R.load_library().rd_basis_create(ctx.h, R._dt(dt), n, cfg.k, nrhs, U0c.data_ptr(), X0.data_ptr(),
                                                  cfg.cap, R.DEVICE, C.byref(h)))
        return h

    L = R.load_library()
    logbuf = np.zeros((nrhs, 5))

    def step(bh, i, host: bool, Xdev=None, Xhost=None):
        its, app = C.c_long(), C.c_long()
        if host:
            hD, hm, sh = pin[i]
            R._check(L.rd_op_set_fields(op.h, hD.data_ptr(), hm.data_ptr(), sh, R.HOST))
            R._check(L.rd_process_system(bh, op.h, nrhs, R._p(idx), R._p(val), cfg.tol, i + 1, 0,
                                         Xhost.ctypes.data_as(C.c_void_p), R.HOST, R._p(logbuf), C.byref(its),
                                         C.byref(app)))
        else:
            set_dev(op, i)
            R._check(L.rd_process_system(bh, op.h, nrhs, R._p(idx), R._p(val), cfg.tol, i + 1, 0,
                                         Xdev.data_ptr(), R.DEVICE, R._p(logbuf), C.byref(its), C.byref(app)))
        rows = logbuf.copy()
        return rows, its.value, app.value

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    # ---- run A: device-resident inputs (value) -----------------------------
    Xdev = torch.empty((nrhs, n), dtype=tdt, device=f"cuda:{local}")
    bh = new_basis()
    sys_ms = []
    for i in range(args.warmup):
        ctx.mark()
        rows, its, app = step(bh, i, host=False, Xdev=Xdev)
        ctx.mark()
        sys_ms.append(ctx.elapsed_ms())
        log(f"warmup system {i + 1}: {sys_ms[-1]:.0f} ms, {its} its, {app} appends, "
            f"{int((rows[:, 3] == 0).sum())} zero-it rows, cols={L.rd_basis_cols(bh)}")
    launches0 = ctx.launches
    ctx.profile(True)
    solves = its_tot = zeros = 0
    barrier()
    torch.cuda.nvtx.range_push("timed")
    with ClockSampler(local) as clk:
        ctx.mark()
        for i in range(args.warmup, args.warmup + args.steps):
            rows, its, app = step(bh, i, host=False, Xdev=Xdev)
            log(f"timed system {i + 1}: {its} its, {app} appends, cols={L.rd_basis_cols(bh)}")
            solves += int((rows[:, 3] > 0).sum())
            zeros += int((rows[:, 3] == 0).sum())
            its_tot += its
        ctx.mark()
        barrier()
    torch.cuda.nvtx.range_pop()
    t_val_ms = ctx.elapsed_ms()
    launches = ctx.launches - launches0
    prof = ctx.prof()
    ctx.profile(False)
    cols_after = L.rd_basis_cols(bh)
    L.rd_basis_destroy(bh)

    # mean per-RHS recycle width over the timed steps (for the CPU sample)
    width = cfg.k + 1 + max(0, (cols_after - cfg.k - nrhs) // max(1, nrhs))

    # ---- run B: end to end through the C ABI with host buffers ------------
    e2e = None
    if not args.no_e2e:
        Xhost = torch.empty((nrhs, n), dtype=tdt).pin_memory().numpy()
        bh = new_basis()
        for i in range(args.warmup):
            step(bh, i, host=False, Xdev=Xdev)
        barrier()
        ctx.mark()
        s2 = 0
        for i in range(args.warmup, args.warmup + args.steps):
            rows, its, app = step(bh, i, host=True, Xhost=Xhost)
            s2 += int((rows[:, 3] > 0).sum())
        ctx.mark()
        barrier()
        t_e2e_ms = ctx.elapsed_ms()
        L.rd_basis_destroy(bh)
        e2e = {"value": s2 / (t_e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * n * 8,
               "d2h_bytes_per_step": n * nrhs * es + nrhs * 5 * 8, "ms": t_e2e_ms}

    # ---- multi-rank aggregation (replicas) ---------------------------------
    t_max, solves_all = t_val_ms, solves
    if dist is not None:
        solves_all, t_max, te = aggregate_replicas(dist, f"cuda:{local}", solves, t_val_ms,
                                                   e2e["ms"] if e2e is not None else None)
        if e2e is not None:
            e2e["value"] = solves_all / (te / 1e3)
    value = solves_all / (t_max / 1e3) if t_max > 0 else 0.0

    # ---- roofline from the live samples ------------------------------------
    def ncu_traffic(kernel, alg_bytes):
        """DRAM read + write per launch for this kernel class from the committed
        ncu --set full capture (profiles/ncu_traffic_r01c.json), scaled from that
        capture's launch to this run's algorithmic bytes per launch."""
        try:
            ref = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                              "ncu_traffic_r01c.json")))
            k = ref["kernels"][kernel]
            ratio = (k["dram_read_bytes"] + k["dram_write_bytes"]) / k["algorithmic_bytes"]
            return round(alg_bytes * ratio), round(ratio, 4), k.get("source", ref["source"])
        except Exception:
            return None, None, None

    peak, peak_kind = measured_peak_hbm()
    classes = {}
    for name, (ms, by, ns) in prof.items():
        if ns:
            classes[name] = {"ms_per_launch": ms / ns, "GBps": by / (ms / 1e3) / 1e9, "samples": ns,
                             "bytes_per_launch": by / ns}
    proj = [k for k in ("ts_T", "ts_NT", "cg_update") if k in classes]
    dominant = max(classes, key=lambda k: prof[k][0]) if classes else None
    roofline = None
    if dominant:
        ach = classes[dominant]["GBps"]
        roofline = {"bound": "hbm", "kernel": dominant, "achieved": round(ach, 1), "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": round(ach / peak, 4),
                    "per_class": classes}
        tr, ratio, src = ncu_traffic(dominant, classes[dominant]["bytes_per_launch"])
        roofline["traffic"] = tr
        roofline["traffic_unit"] = "bytes per launch (DRAM read + write)"
        roofline["traffic_over_algorithmic"] = ratio
        roofline["traffic_source"] = src
        if proj:
            tot_ms = sum(prof[k][0] for k in proj)
            tot_b = sum(prof[k][1] for k in proj)
            roofline["projections_combined_GBps"] = round(tot_b / (tot_ms / 1e3) / 1e9, 1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            mean_its = its_tot / max(1, solves)
            cs = cpu_sample(cfg, width, mean_its, args.cpu_iters)
            cpu = {"value": cs["value"], "unit": UNIT, "cores": host_cores(), "kind": "port",
                   "sample": cs["sample"], "t_from_raw_s": cs["t_from_raw_s"], "t_iter_s": cs["t_iter_s"]}
        except Exception as e:  # the baseline must never sink the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "c128" if cfg.complex else "f64", "data": "synthetic (seeded Gaussian-RBF level sets)",
            "config": {"workload": f"{cfg.name}: {g.d}D {g.N[0]}^{g.d} (n={n}), {nrhs} RHS, k={cfg.k}, "
                                   f"omega/nu in {list(cfg.omegas)}, tol={cfg.tol}, cap={cfg.cap}",
                       "step": "one process_system (one parameter point x frequency system)",
                       "systems_timed": [list(s) for s in systems[args.warmup:]],
                       "l2": "inputs larger than L2 (basis n x r streamed every iteration)",
                       "parallelism": f"replicas x{world}"},
            "solves": solves, "zero_iteration_rhs": zeros, "inner_iterations": its_tot,
            "iterations_per_s": its_tot / (t_val_ms / 1e3) if t_val_ms else 0.0,
            "basis_cols": cols_after,
            "seed_s": {"eigenpairs_U0": t_eig, "X0_solves": t_x0, "X0_iterations": tot.value},
            "warmup_system_ms": sys_ms,
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clk.summary(), "field_gen_s": t_gen,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args, cfg, world, rank):
    """--impl reference: the CPU oracle (restatement of the reference's CPU
    path; the reference itself cannot be built here) on the box's host cores,
    each step a bounded sample of the same workload."""
    if rank != 0:
        return
    cores = host_cores()
    os.environ["OMP_NUM_THREADS"] = str(cores)
    # the device arm's measured workload at the same timed systems (4-5) of C4
    # (profiles/r01g_bench_c4.json): recycle width k + 1 + ~4 own appends,
    # 11,286 inner iterations over 128 solves
    width = cfg.k + 1 + 4
    mean_its = 88.2
    vals = []
    t0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        cs = cpu_sample(cfg, width, mean_its, args.cpu_iters)
        if i >= args.warmup:
            vals.append(cs["value"])
    dt = time.perf_counter() - t0
    v = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128" if cfg.complex else "f64",
            "data": "synthetic", "config": {"workload": cfg.name, "parallelism": "cpu"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": cs["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": dt}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
