import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as rd
c = P.CONFIGS["T2c"]; g, lay = c.grid, c.layout()
z = np.load("tests/golden/T2c.npz") if False else None
f0 = c.fields(0)
lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, 1e-8)
X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
U0 = U0.astype(c.dtype)
rep = int(sys.argv[1])
for r in range(rep):
    gb = rd.GlobalBasis(U0, X0, c.cap)
    for s,(pt,w) in enumerate(c.systems(), start=1):
        sys.stderr.write(f"=== rep {r} system {s}\n")
        rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
