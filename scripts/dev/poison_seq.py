"""ROMDOT_POISON=1 hunt: T2 build then T2c build in one process (the order that trips the
poisoned-allocation check), every solution checked for NaN."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as rd
for name in sys.argv[1:] or ["T2", "T2c"]:
    c = P.CONFIGS[name]; g, lay = c.grid, c.layout()
    f0 = c.fields(0)
    lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, min(c.tol, 1e-8))
    X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    gb = rd.GlobalBasis(U0.astype(c.dtype), X0, c.cap)
    for s, (pt, w) in enumerate(c.systems(), start=1):
        print(f"#### {name} system {s}", file=sys.stderr, flush=True)
        pr = rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
        bad = [j for j in range(lay.n_rhs) if not np.isfinite(pr.X[:, j]).all()]
        print(name, s, "cols", gb.cols, "its", pr.inner_iterations, "nan columns", bad, flush=True)
