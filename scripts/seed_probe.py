"""Time the device eigen seed (U0) and one X0 solve on a config (diagnostics)."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_00138_b200 import build, problem as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--k", type=int, default=0)
    args = ap.parse_args()
    build.build()
    from paper_1602_00138_b200 import romdot as R
    cfg = P.CONFIGS[args.config]
    g, lay = cfg.grid, cfg.layout()
    f0 = cfg.fields(0)
    k = args.k or cfg.k
    op_r = R.SchurOperator(g, f0, np.float64)
    b = np.zeros(g.n)
    b[lay.idx[0]] = lay.val[0]
    t0 = time.perf_counter()
    res = R.recycled_cg(op_r, None, None, b, 0.25 * cfg.tol, 2 * g.n)
    print(f"one real CG solve: {res.report.iterations} its, {time.perf_counter() - t0:.2f}s, relres {res.report.final_relres:.2e}", flush=True)
    t0 = time.perf_counter()
    res = R.recycled_cg(op_r, None, None, b, 1e-10, 2 * g.n)
    print(f"one real CG solve at 1e-10: {res.report.iterations} its, {time.perf_counter() - t0:.2f}s", flush=True)
    t0 = time.perf_counter()
    lam, U = R.smallest_eigenpairs(op_r, k, min(cfg.tol, 1e-8))
    print(f"eigenpairs k={k}: {time.perf_counter() - t0:.2f}s lam[:4]={lam[:4]}", flush=True)


if __name__ == "__main__":
    main()
