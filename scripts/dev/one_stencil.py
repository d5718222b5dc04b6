import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1602_00138_b200 import problem as P, romdot as R
d, N, cplx, nc = int(sys.argv[1]), tuple(int(v) for v in sys.argv[2].split(",")), sys.argv[3] == "c", int(sys.argv[4])
g = P.GridSpec(d=d, N=N, h=1.0 / (N[0] - 1), D_bg=0.33)
rng = np.random.default_rng(5)
f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=g.h ** 2 * rng.uniform(0.005, 0.05, g.n), shift=0.01 if cplx else 0.0)
dt = np.complex128 if cplx else np.float64
x = rng.standard_normal((g.n, nc)) + (1j * rng.standard_normal((g.n, nc)) if cplx else 0)
op = R.SchurOperator(g, f, dt)
y = op.apply(x)
y1 = np.stack([op.apply(np.ascontiguousarray(x[:, j])) for j in range(nc)], axis=1)
print(sys.argv[1:], "max diff", np.abs(y - y1).max(), flush=True)
