import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle'); sys.path.insert(0,'tests')
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as rd

def seed(c, g, lay):
    f0 = c.fields(0)
    lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, 1e-8)
    X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    return U0.astype(c.dtype), X0

def run(name):
    c = P.CONFIGS[name]; g, lay = c.grid, c.layout()
    U0, X0 = seed(c, g, lay)
    gb = rd.GlobalBasis(U0, X0, c.cap)
    logs = []
    for s,(pt,w) in enumerate(c.systems(), start=1):
        pr = rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
        logs += [(r.init_relres, r.iterations) for r in pr.log]
    return np.array(logs), gb.V

for name in ["T2", "T2c", "T3c", "T2c", "T2c"]:
    l, V = run(name)
    print(name, l[-3:, 0], V.shape, abs(V).sum())
a = [run("T2c") for _ in range(3)]
for i in range(1, 3):
    print("T2c rerun identical:", np.array_equal(a[0][0], a[i][0]), a[0][1].tobytes() == a[i][1].tobytes(),
          np.abs(a[0][0][:,0]-a[i][0][:,0]).max())
