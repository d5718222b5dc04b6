"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck /
initcheck): every kernel family of the library on tiny shapes -- device seed,
batched X0 CG, a T3c build (fused one-launch CG iteration cg_fused, TMA
projections, refresh / append / per-RHS spaces, cap), the TMA multi-column
stencil (complex odd N0 through the padded fields, real even N0), the RRQR
and the reduced model. Run by scripts/sanitize.sh; prints "sanitize ok".
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_00138_b200 import problem as P  # noqa: E402
from paper_1602_00138_b200 import romdot as R  # noqa: E402


def main():
    c = P.CONFIGS["T3c"]
    g, lay = c.grid, c.layout()
    f0 = c.fields(0)
    lam, U0 = R.smallest_eigenpairs(R.SchurOperator(g, f0, np.float64), c.k, 1e-8)
    X0, _ = R.initial_solutions(R.SchurOperator(g, f0, c.dtype), lay, c.tol)
    gb = R.GlobalBasis(U0.astype(c.dtype), X0, c.cap)
    for s, (pt, w) in enumerate(c.systems(), start=1):
        pr = R.process_system(gb, R.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
        res = R.residual_norms(R.SchurOperator(g, c.fields(pt, w), c.dtype), lay, pr.X)
        assert res.max() <= c.tol, res.max()
    rank, _, _ = gb.compress(1e-10)
    rom = R.ReducedModel(gb.V)
    psi = rom.transfer(R.SchurOperator(g, c.fields(1, 0.1), c.dtype), lay)
    assert np.isfinite(psi).all()
    for d, N, cplx in [(3, (11, 9, 13), True), (3, (12, 10, 6), False), (2, (37, 29), True)]:
        gs = P.GridSpec(d=d, N=N, h=1.0 / (N[0] - 1), D_bg=0.33)
        rng = np.random.default_rng(1)
        fs = P.Fields(D=rng.uniform(0.3, 0.4, gs.n), mu=gs.h ** 2 * rng.uniform(0.005, 0.05, gs.n),
                      shift=0.01 if cplx else 0.0)
        x = rng.standard_normal((gs.n, 9))
        if cplx:
            x = x + 1j * rng.standard_normal((gs.n, 9))
        R.SchurOperator(gs, fs, np.complex128 if cplx else np.float64).apply(x)
    A = np.random.default_rng(2).standard_normal((4000, 40)) * (0.9 ** np.arange(40))
    R.rrqr(A, 1e-10)
    print(f"sanitize ok: rank {rank}, cols {gb.cols}")


if __name__ == "__main__":
    main()
