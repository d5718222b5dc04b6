import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle'); sys.path.insert(0,'tests')
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as rd
HERE='tests/golden'
def golden_build(name):
    z = np.load(f"{HERE}/{name}.npz"); c = P.CONFIGS[name]; g, lay = c.grid, c.layout()
    gb = rd.GlobalBasis(z["U0"], z["X0"], c.cap)
    for s,(pt,w) in enumerate(c.systems(), start=1):
        rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s, want_X=False)
c = P.CONFIGS["T2c"]; g, lay = c.grid, c.layout()
f0 = c.fields(0)
lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, 1e-8)
X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
U0 = U0.astype(c.dtype)
ref = None
for rep in range(12):
    if rep % 3 == 1: golden_build("T2"); golden_build("T3c")
    gb = rd.GlobalBasis(U0, X0, c.cap)
    rows = []; Vs = []
    for s,(pt,w) in enumerate(c.systems(), start=1):
        pr = rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
        rows += [(s, r.rhs, r.init_relres, r.iterations) for r in pr.log]
        Vs.append(gb.V.copy())
    rows = np.array(rows)
    if ref is None:
        ref = (rows, Vs); print("rep0 ok"); continue
    d = np.abs(rows[:,2] - ref[0][:,2]) / ref[0][:,2]
    bad = np.nonzero(d > 1e-13)[0]
    vd = [np.abs(a - b).max() for a, b in zip(Vs, ref[1])]
    print(f"rep {rep}: first diff row {bad[:1]} (sys,rhs)={rows[bad[0],:2] if len(bad) else None} maxrel {d.max():.2e} its diff {np.abs(rows[:,3]-ref[0][:,3]).max()} Vdiff per system {['%.1e'%v for v in vd]}")
