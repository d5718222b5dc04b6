"""Full-configuration parity of the device basis build against the CPU
checker (north_star tolerances) on a BASELINE config whose
oracle run finishes in minutes (default C1):

* lockstep: both builds from the same (oracle) seed U0 / X0, system by system;
  every BuildLog row compared (append decision, iterations +/-2, init_relres),
  every device solution's explicit residual <= tol;
* compression: RRQR at 1e-10 of both candidate bases -> same retained rank,
  largest principal-angle sine between the compressed bases <= 1e-6;
* observables: reduced transfer and Jacobian (device ReducedModel on each
  compressed basis, same code) at an off-training parameter point, <= 1e-8
  relative.

Prints one JSON line (saved under profiles/ by the caller).

At the target config (C4, n = 2,097,152 complex) the CPU checker cannot run
the whole build in a GPU call (~35 s per solve on 16 host cores), so
``--rhs m --device-seed`` runs the same lockstep on the first m RHS of the
first systems, seeded with the DEVICE U0 / X0 (checked here against the
checker's operator: eigen-residuals and X0 explicit residuals), and the
compression and observable checks on the resulting candidate bases.
Free-running builds can diverge after an append-decision flip on a marginal
RHS; the lockstep comparison reports the flips it sees.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1602_00138_b200 import build, problem as P  # noqa: E402


def principal_sines(Q1, Q2):
    """sin of the principal angles between span(Q1) and span(Q2) (orthonormal)."""
    s = np.linalg.svd(Q1.conj().T @ Q2, compute_uv=False)
    s = np.clip(s, 0.0, 1.0)
    return np.sqrt(np.maximum(0.0, 1.0 - s * s))


def run(config: str, n_systems: int = 0, n_rhs: int = 0, device_seed: bool = False) -> dict:
    import oracle as orc
    from paper_1602_00138_b200 import romdot as R
    c = P.CONFIGS[config]
    g, lay_full = c.grid, c.layout()
    lay = lay_full
    if n_rhs:  # first n_rhs right-hand sides of every system (the basis keeps all X0 columns)
        lay = P.Layout(lay_full.idx[:n_rhs].copy(), lay_full.val[:n_rhs].copy(), min(n_rhs, lay_full.n_src),
                       max(0, n_rhs - lay_full.n_src))
    t0 = time.perf_counter()
    f0 = c.fields(0)
    seed_check = {}
    if device_seed:
        lam, U0 = R.smallest_eigenpairs(R.SchurOperator(g, f0, np.float64), c.k, min(c.tol, 1e-8))
        X0, _ = R.initial_solutions(R.SchurOperator(g, f0, c.dtype), lay_full, c.tol)
        # the device seed, checked with the checker's own operator
        op_r = orc.Operator.grid(g, f0)
        er = np.linalg.norm(op_r.apply(U0) - U0 * lam, axis=0)
        seed_check["eig_residual_over_lammax"] = float(er.max() / op_r.lam_max)
        op0 = orc.Operator.grid(g, f0, c.dtype)
        B0 = lay_full.dense(g.n, c.dtype)
        seed_check["X0_max_explicit_residual"] = float(
            (np.linalg.norm(op0.apply(X0) - B0, axis=0) / np.linalg.norm(B0, axis=0)).max())
        del B0
    else:
        lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, min(c.tol, 1e-8))
        X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    U0 = U0.astype(c.dtype)
    t_seed = time.perf_counter() - t0
    gb_o = orc.GlobalBasis(U0, X0, c.cap)
    gb_g = R.GlobalBasis(U0, X0, c.cap)
    del U0, X0
    systems = c.systems()[: n_systems] if n_systems else c.systems()
    rows = flips = worst_its = 0
    worst_relres = worst_res = worst_res_cpu = xdiff = 0.0
    log_rows = []
    t_cpu = t_gpu = 0.0
    B = lay.dense(g.n, c.dtype)
    for s, (pt, w) in enumerate(systems, start=1):
        f = c.fields(pt, w)
        op_o = orc.Operator.grid(g, f, c.dtype)
        t0 = time.perf_counter()
        po = orc.process_system(gb_o, op_o, lay, c.tol, s)
        t_cpu += time.perf_counter() - t0
        t0 = time.perf_counter()
        pg = R.process_system(gb_g, R.SchurOperator(g, f, c.dtype), lay, c.tol, s)
        t_gpu += time.perf_counter() - t0
        res = np.linalg.norm(op_o.apply(pg.X) - B, axis=0) / np.linalg.norm(B, axis=0)
        worst_res = max(worst_res, float(res.max()))
        res_o = np.linalg.norm(op_o.apply(po.X) - B, axis=0) / np.linalg.norm(B, axis=0)
        worst_res_cpu = max(worst_res_cpu, float(res_o.max()))
        xdiff = max(xdiff, float((np.linalg.norm(pg.X - po.X, axis=0) / np.linalg.norm(po.X, axis=0)).max()))
        log_rows += [[s, ro.rhs, ro.iterations, rg.iterations, ro.init_relres, rg.init_relres, int(ro.appended),
                      int(rg.appended)] for ro, rg in zip(po.log, pg.log)]
        for ro, rg in zip(po.log, pg.log):
            rows += 1
            if ro.appended != rg.appended:
                flips += 1
                continue
            worst_its = max(worst_its, abs(ro.iterations - rg.iterations))
            if ro.init_relres > 0:
                worst_relres = max(worst_relres, abs(ro.init_relres - rg.init_relres) / ro.init_relres)
        del po, pg
        print(json.dumps({"system": s, "cols_cpu": gb_o.cols, "cols_gpu": gb_g.cols, "flips": flips}),
              file=sys.stderr, flush=True)
        if flips:
            break
    print(json.dumps({"lockstep_rows": rows, "append_flips": flips, "max_iteration_diff": worst_its,
                      "max_init_relres_reldiff": worst_relres, "max_explicit_residual_gpu": worst_res,
                      "max_explicit_residual_cpu": worst_res_cpu, "max_solution_reldiff": xdiff, **seed_check}),
          file=sys.stderr, flush=True)
    # compression: RRQR of each candidate basis at 1e-10 (normalised columns)
    Vo = gb_o.V
    rank_o, _, _, Qo = orc.qrcp(Vo, 1e-10, True)
    rank_g, _, _ = gb_g.compress(1e-10)
    Qg = gb_g.V
    sines = principal_sines(Qo[:, :rank_o], Qg[:, :rank_g]) if rank_o == rank_g else np.array([1.0])
    # observables at an off-training point (the next point of the sequence)
    npt = c.n_points + 1
    f = c.fields(npt, c.omegas[-1])
    op = R.SchurOperator(g, f, c.dtype)
    rom_o = R.ReducedModel(Qo[:, :rank_o])
    rom_g = R.ReducedModel(Qg[:, :rank_g])
    psi_o, psi_g = rom_o.transfer(op, lay_full), rom_g.transfer(op, lay_full)
    rng = np.random.default_rng(7)
    sup = [(np.sort(rng.choice(g.n, size=g.n // 20, replace=False)), rng.uniform(0.1, 1.0, g.n // 20))
           for _ in range(4)]
    J_o = rom_o.jacobian(op, lay_full, sup, -g.h ** 2)
    J_g = rom_g.jacobian(op, lay_full, sup, -g.h ** 2)
    fom, _ = R.fom_transfer(op, lay_full, 1e-10)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    out = {"config": config, "systems": len(systems), "rows": rows, "append_flips": flips,
           "max_iteration_diff": worst_its, "max_init_relres_reldiff": worst_relres,
           "max_explicit_residual_gpu": worst_res, "max_explicit_residual_cpu": worst_res_cpu,
           "max_solution_reldiff": xdiff, "tol": c.tol, "rhs_per_system": lay.n_rhs,
           "seed": "device (checked with the checker's operator)" if device_seed else "checker", **seed_check,
           "log_cpu_vs_gpu": log_rows if n_rhs else None,
           "rank_cpu": int(rank_o), "rank_gpu": int(rank_g), "max_principal_sine": float(sines.max()),
           "rom_transfer_reldiff": rel(psi_g, psi_o), "rom_jacobian_reldiff": rel(J_g, J_o),
           "rom_vs_fom_offtraining": rel(psi_g, fom),
           "pass": bool(flips == 0 and worst_its <= 2 and worst_res <= c.tol and rank_o == rank_g
                        and sines.max() <= 1e-6 and rel(psi_g, psi_o) <= 1e-8 and rel(J_g, J_o) <= 1e-8),
           "cpu_s": round(t_cpu, 2), "gpu_s": round(t_gpu, 2), "seed_s_cpu": round(t_seed, 2)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--systems", type=int, default=0)
    ap.add_argument("--rhs", type=int, default=0, help="first m RHS per system (0 = all)")
    ap.add_argument("--device-seed", action="store_true", help="U0 / X0 from the device (checked), not the checker")
    args = ap.parse_args()
    build.build()
    print(json.dumps(run(args.config, args.systems, args.rhs, args.device_seed)))


if __name__ == "__main__":
    main()
