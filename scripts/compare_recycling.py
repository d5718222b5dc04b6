"""cmd_compare_recycling (harness.cpp:209-252, acceptance criterion 5) on the
B200: the global-basis build (process_system) and the per-RHS-only
comparator (BaselinePerRhsRecycler) from the same device seed, the reference's
first min(K, 2) systems by default. Prints one JSON line with the inner
iteration totals, the ratio and the device time of each."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_00138_b200 import build, problem as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--systems", type=int, default=2, help="0 = all (the reference uses min(K, 2))")
    args = ap.parse_args()
    build.build()
    from paper_1602_00138_b200 import romdot as R
    c = P.CONFIGS[args.config]
    g, lay = c.grid, c.layout()
    op0r = R.SchurOperator(g, c.fields(0), np.float64)
    op0 = R.SchurOperator(g, c.fields(0), c.dtype)
    lam, U0 = R.smallest_eigenpairs(op0r, c.k, min(c.tol, 1e-8))
    X0, _ = R.initial_solutions(op0, lay, c.tol)
    gb = R.GlobalBasis(U0.astype(c.dtype), X0, c.cap)
    pr = R.PerRhsRecycler(U0.astype(c.dtype), X0)
    systems = c.systems()[: args.systems] if args.systems else c.systems()
    ours = base = 0
    t_ours = t_base = 0.0
    zero_ours = zero_base = 0
    rows = []
    for s, (pt, w) in enumerate(systems, start=1):
        f = c.fields(pt, w)
        op = R.SchurOperator(g, f, c.dtype)
        t0 = time.perf_counter()
        a = R.process_system(gb, op, lay, c.tol, s, want_X=False)
        t_ours += time.perf_counter() - t0
        t0 = time.perf_counter()
        b = pr.solve_system(op, lay, c.tol, s, want_X=False)
        t_base += time.perf_counter() - t0
        ours += a.inner_iterations
        base += b.inner_iterations
        zero_ours += sum(r.iterations == 0 for r in a.log)
        zero_base += sum(r.iterations == 0 for r in b.log)
        rows.append({"system": s, "its_ours": a.inner_iterations, "its_baseline": b.inner_iterations})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"config": args.config, "systems": len(systems), "n_rhs": lay.n_rhs, "ours": ours,
                      "baseline": base, "ratio": ours / max(base, 1), "criterion5_pass": ours > 0 and 2 * ours <= base,
                      "zero_iteration_rhs_ours": zero_ours, "zero_iteration_rhs_baseline": zero_base,
                      "ours_s": round(t_ours, 3), "baseline_s": round(t_base, 3), "per_system": rows}))


if __name__ == "__main__":
    main()
