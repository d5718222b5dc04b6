"""Checkpoint-replay lockstep over a whole BASELINE build (default C4, all 16
systems): the device builds, the CPU checker replays sampled RHS from the
device's state (oracle/replay.py). Prints one JSON object (saved under
profiles/ by the caller).

  python scripts/c4_replay.py --config C4 --per-system 2 --gram 16
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1602_00138_b200 import build, problem as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--per-system", type=int, default=2)
    ap.add_argument("--systems", type=int, default=0, help="first m systems (0 = all)")
    ap.add_argument("--factor", default="1,2,9,10,16", help="systems whose refresh factor is checked")
    ap.add_argument("--gram", default="16", help="systems whose full K_img^H K_img is checked")
    args = ap.parse_args()
    build.build()
    import replay as RP
    c = P.CONFIGS[args.config]
    lay = c.layout()
    ns = args.systems or len(c.systems())
    pts = RP.default_points(ns, lay.n_rhs, lay.n_src, args.per_system)
    fac = [int(s) for s in args.factor.split(",") if s and int(s) <= ns]
    gram = [int(s) for s in args.gram.split(",") if s and int(s) <= ns]
    t0 = time.perf_counter()
    out, smp = RP.run_device_build(c, pts, systems=list(range(1, ns + 1)), factor_check_systems=fac,
                                   gram_check_systems=gram)
    out["config"] = args.config
    out["tol"] = c.tol
    out["points"] = {str(k): sorted(v) for k, v in pts.items()}
    out["host_cores"] = os.cpu_count()
    out["wall_s"] = time.perf_counter() - t0
    out["pass"] = bool(out["append_flips"] == 0 and out["max_iteration_diff"] <= 2
                       and out["max_init_relres_reldiff"] <= 1e-6 and out["max_solution_reldiff"] <= 1e-6
                       and out["max_explicit_residual_gpu"] <= c.tol and out["all_converged"]
                       and all(f["KR_minus_AV_rel"] <= 1e-12 and f.get("KhK_minus_I_max", 0) <= 1e-11
                               for f in out["factor_checks"].values()))
    # K_img^H K_img = I is checked entrywise at 1e-11: the one-pass CholQR
    # refresh (second pass only when kappa_1(S) > 20) leaves ~kappa^2 eps of
    # non-orthogonality, 1.8e-12 at r = 768 (profiles/r02_c4_replay.json)
    out["bars"] = {"KR_minus_AV_rel": 1e-12, "KhK_minus_I_max": 1e-11, "iterations": 2, "init_relres": 1e-6,
                   "solution": 1e-6, "explicit_residual": c.tol}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
