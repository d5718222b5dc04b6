"""Batched tail (ROMDOT_BATCH=1) against the one-solve path (ROMDOT_BATCH=0) on a capped config."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1602_00138_b200 import problem as P, romdot as rd

N = int(os.environ.get("PN", "48")); k = int(os.environ.get("PK", "64")); cplx = int(os.environ.get("PC", "1"))
ns = (4, 6)
cfg = P.ProblemConfig("probe", d=3, N=N, n_src=ns, n_det=ns, m_rbf=6, n_points=int(os.environ.get("PP", "3")), omegas=(0.0, 0.1) if cplx else (0.0,),
                      k=k, complex=bool(cplx), cap=k + 48 + int(os.environ.get("PCAP", "30")))
g, lay = cfg.grid, cfg.layout()
ctx = rd.Context(0)
f0 = cfg.fields(0)
op0r = rd.SchurOperator(g, f0, np.float64, ctx)
lam, U0 = rd.smallest_eigenpairs(op0r, cfg.k, 1e-8)
op0 = rd.SchurOperator(g, f0, cfg.dtype, ctx)
X0, _ = rd.initial_solutions(op0, lay, cfg.tol)
res = {}
for mode in os.environ.get("MODES", "0,1").split(","):
    os.environ["ROMDOT_BATCH"] = mode
    gb = rd.GlobalBasis(U0.astype(cfg.dtype), X0, cfg.cap, ctx)
    op = rd.SchurOperator(g, f0, cfg.dtype, ctx)
    out = []
    for s, (pt, w) in enumerate(cfg.systems(), start=1):
        op.set_fields(cfg.fields(pt, w))
        prof = int(os.environ.get("PROF_SYS", "0")) == s
        if prof:
            import torch
            torch.cuda.synchronize(); torch.cuda.profiler.start()
        ctx.sync(); t0 = time.time()
        pr = rd.process_system(gb, op, lay, cfg.tol, s)
        ctx.sync(); dt = time.time() - t0
        if prof:
            torch.cuda.synchronize(); torch.cuda.profiler.stop()
        rn = rd.residual_norms(op, lay, pr.X)
        out.append((pr, dt, rn.max()))
        print(f"mode {mode} system {s}: cols {gb.cols} its {pr.inner_iterations} appended {sum(r.appended for r in pr.log)} "
              f"time {dt*1e3:.0f} ms maxres {rn.max():.2e}", flush=True)
    res[mode] = out
for (a, _, _), (b, _, _) in (zip(res["0"], res["1"]) if len(res) == 2 else []):
    ia = np.array([r.iterations for r in a.log]); ib = np.array([r.iterations for r in b.log])
    fa = [r.appended for r in a.log]; fb = [r.appended for r in b.log]
    ra = np.array([r.init_relres for r in a.log]); rb = np.array([r.init_relres for r in b.log])
    print("its diff", (ib - ia).min(), (ib - ia).max(), "flags", fa == fb, "init_relres", np.abs(rb / ra - 1).max(),
          "X", np.linalg.norm(a.X - b.X) / np.linalg.norm(a.X))
