import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as rd
for name, width in [("T2c", 9), ("T2c", 13), ("T2", 9), ("T3c", 12)]:
    c = P.CONFIGS[name]; g, lay = c.grid, c.layout()
    pt, w = c.systems()[-1]
    f = c.fields(pt, w)
    op_o = orc.Operator.grid(g, f, c.dtype)
    rng = np.random.default_rng(11)
    W = rng.standard_normal((g.n, width)).astype(c.dtype)
    rs = orc.RecycleSpace(W, op_o.apply(W))
    U, K = rs.UK()
    b = lay.dense(g.n, c.dtype)[:, 0]
    _, r0 = rs.initial_guess(b)
    op = rd.SchurOperator(g, f, c.dtype)
    outs = []
    for rep in range(60):
        res = rd.recycled_cg(op, U, K, r0, 1e-9, 2 * g.n, np.linalg.norm(b))
        outs.append((res.report.iterations, res.correction.copy()))
    its = [o[0] for o in outs]
    diffs = [np.abs(o[1] - outs[0][1]).max() for o in outs]
    print(name, width, "its set", sorted(set(its)), "max diff", max(diffs), "n nonzero diffs", sum(d > 0 for d in diffs))
