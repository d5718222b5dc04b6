"""Kernels for one `ncu --set full` capture each (run under ncu with -k):
the TMA multi-column stencil at the C4 refresh shape (768 columns), the DMMA
Gram (V^H V, 768 complex columns), the DMMA tall GEMM (768 x 768 complex) and
the RRQR of the C5 0.9-decay matrix (n = 2M, m = 1024, real)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1602_00138_b200 import problem as P, romdot as R  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
ctx = R.default_context()
if what in ("all", "stencil"):
    g = P.CONFIGS["C4"].grid
    rng = np.random.default_rng(5)
    f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=g.h ** 2 * rng.uniform(0.005, 0.05, g.n), shift=g.h ** 2 * 0.1)
    op = R.SchurOperator(g, f, np.complex128)
    print("stencil 768 ms", R.bench_stencil(op, 768, 2))
if what in ("all", "gram"):
    print("gram c128 768 ms", R.bench_gram(2097152, 768, 768, True, True, iters=1, ctx=ctx))
if what in ("all", "gemm"):
    print("gemm c128 768 ms", R.bench_gemm(2097152, 768, 768, True, upper=False, iters=1, ctx=ctx))
