"""Regenerate the committed golden fixtures (CPU oracle, deterministic).

For each small parity config: the seed (U0 from the oracle's shift-invert
Lanczos, X0 from oracle CG at 0.25 tol), the full BuildLog of every system,
the final basis width and the reduced transfer function at the last system.
Run:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as orc  # noqa: E402
from helpers import rom_transfer  # noqa: E402
from paper_1602_00138_b200 import problem as P  # noqa: E402

CONFIGS = ["T2", "T3c"]


def make(name):
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    f0 = c.fields(0)
    lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, min(c.tol, 1e-8))
    U0 = U0.astype(c.dtype)
    X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    gb = orc.GlobalBasis(U0, X0, c.cap)
    logs = []
    op = None
    for s, (pt, w) in enumerate(c.systems(), start=1):
        op = orc.Operator.grid(g, c.fields(pt, w), c.dtype)
        pr = orc.process_system(gb, op, lay, c.tol, s)
        logs += [[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in pr.log]
    B = lay.dense(g.n, c.dtype)
    psi = rom_transfer(gb.V, op.matrix(), B[:, : lay.n_src], B[:, lay.n_src:])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), U0=U0, X0=X0, lam=lam, log=np.array(logs),
                        cols=gb.cols, psi=psi)
    print(name, "cols", gb.cols, "rows", len(logs))


if __name__ == "__main__":
    for n in CONFIGS:
        make(n)
