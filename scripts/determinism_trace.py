"""Run interleaved T3c/T2c builds with ROMDOT_VERBOSE=4 (async device hash log);
markers go to stderr so the log can be split per build. Compare with
scripts/determinism_trace_cmp.py <log>."""
import sys
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as rd
def seed(name):
    c = P.CONFIGS[name]; g, lay = c.grid, c.layout()
    f0 = c.fields(0)
    lam, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, 1e-8)
    X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    return U0.astype(c.dtype), X0
S = {n: seed(n) for n in ["T2c", "T3c"]}
def build(name, rep):
    c = P.CONFIGS[name]; g, lay = c.grid, c.layout()
    gb = rd.GlobalBasis(*S[name], c.cap)
    for s,(pt,w) in enumerate(c.systems(), start=1):
        sys.stderr.write(f"=== {name} rep {rep} system {s}\n"); sys.stderr.flush()
        rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
for r in range(int(sys.argv[1])):
    build("T3c", r)
    build("T2c", r)
