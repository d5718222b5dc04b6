import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import oracle as orc
from paper_1602_00138_b200 import problem as P, build
build.build()
from paper_1602_00138_b200 import romdot as rd
d, N, cplx, width = 3, (48, 40, 44), True, 20
if len(sys.argv) > 1:
    width = int(sys.argv[1])
g = P.GridSpec(d=d, N=N, h=1.0 / (N[0] - 1), D_bg=0.33)
rng = np.random.default_rng(8)
f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=g.h ** 2 * rng.uniform(0.005, 0.05, g.n), shift=g.h ** 2 * 0.1)
dt = np.complex128
op_o = orc.Operator.grid(g, f, dt)
rng = np.random.default_rng(21)
W = (rng.standard_normal((g.n, width)) + 1j * rng.standard_normal((g.n, width))).astype(dt)
U, K = rd.recycle_space_from_raw(W, op_o.apply(W))
b = rng.standard_normal(g.n).astype(dt)
r0 = b - K @ (K.T @ b)
op_g = rd.SchurOperator(g, f, dt)
H = {}
for fused in ("0", "1", "1"):
    os.environ["ROMDOT_FUSED"] = fused
    res = rd.recycled_cg(op_g, U, K, r0, 1e-9, 2 * g.n, np.linalg.norm(b))
    h = res.report.rel_residual_history
    print(fused, res.report.iterations, res.report.converged, h[-3:])
    H.setdefault(fused, []).append(h)
a, c = H["0"][0], H["1"][0]
m = min(len(a), len(c))
rel = np.abs(c[:m] - a[:m]) / a[:m]
idx = np.argmax(rel > 1e-6) if (rel > 1e-6).any() else -1
print("first divergence > 1e-6 at", idx, a[max(0, idx - 3):idx + 3], c[max(0, idx - 3):idx + 3])
print("fused deterministic:", np.array_equal(H["1"][0], H["1"][1]))
for it in [0, 1, 2, 5, 10, 50, 100, 200, 300, 400, 500]:
    if it < m: print(it, a[it], c[it])
c = H["1"][0]
k = int(np.argmax(c == c[-1]))
print("constant from", k, c[k - 8:k + 3])
