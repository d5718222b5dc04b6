"""Build determinism check with no extra device calls: interleaved T3c/T2c builds,
X hashed per system and V per build; reports the first system whose output differs
from the first build (usage: diag_race3.py REPS)."""
import hashlib, sys, numpy as np
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
H = lambda a: hashlib.md5(np.ascontiguousarray(a).tobytes()).hexdigest()[:8]
def build(name):
    c = P.CONFIGS[name]; g, lay = c.grid, c.layout()
    gb = rd.GlobalBasis(*S[name], c.cap)
    out, Xs = [], []
    for s,(pt,w) in enumerate(c.systems(), start=1):
        pr = rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
        out.append((s, H(pr.X), gb.cols, tuple(r.iterations for r in pr.log), tuple(r.appended for r in pr.log)))
        Xs.append(pr.X)
    out.append(("V", H(gb.V)))
    return out, Xs
ref, Xr = build("T2c")
N = int(sys.argv[1]); bad = 0
for r in range(N):
    build("T3c")
    x, Xx = build("T2c")
    for i, (a, b) in enumerate(zip(x, ref)):
        if a != b:
            bad += 1
            msg = ""
            if i < len(Xx):
                d = np.abs(Xx[i] - Xr[i]).max(0) / np.abs(Xr[i]).max(0)
                msg = "col reldiff " + " ".join(f"{v:.1e}" for v in d)
            print("rep", r, "first diff", a, "ref", b, msg, flush=True)
            break
print("reps", N, "bad", bad)
