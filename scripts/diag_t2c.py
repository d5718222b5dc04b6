import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle'); sys.path.insert(0,'tests')
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as rd
c = P.CONFIGS["T2c"]; g, lay = c.grid, c.layout()
f0 = c.fields(0)
lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, 1e-8)
X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
U0 = U0.astype(c.dtype)
gb_o = orc.GlobalBasis(U0, X0, c.cap); gb_g = rd.GlobalBasis(U0, X0, c.cap)
for s,(pt,w) in enumerate(c.systems(), start=1):
    f = c.fields(pt, w)
    po = orc.process_system(gb_o, orc.Operator.grid(g, f, c.dtype), lay, c.tol, s)
    pg = rd.process_system(gb_g, rd.SchurOperator(g, f, c.dtype), lay, c.tol, s)
    for a,b in zip(po.log, pg.log):
        print(s, a.rhs, f"{a.init_relres:.10e} {b.init_relres:.10e} {abs(a.init_relres-b.init_relres)/a.init_relres:.1e}", a.iterations, b.iterations, a.appended, b.appended)
    K_o = gb_o.K_img; K_g = gb_g.K_img
    print("cols", gb_o.cols, gb_g.cols, "proj diff", np.abs(K_o@K_o.conj().T - K_g@K_g.conj().T).max())
