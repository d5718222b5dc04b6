"""Device MINRES (ctx solver 1) against the reference fixtures: prints the row differences."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1602_00138_b200 import problem as P, romdot as rd

G = os.path.join(ROOT, "tests", "golden")
rel = lambda a, b: float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))
ctx = rd.Context(0)
ctx.set_solver(int(os.environ.get("SOLVER", "1")))
z = np.load(os.path.join(G, "ref_desk.npz"))
n = int(z["n"]); g = P.GridSpec.reference_2d(n, n)
lay = P.make_layout(g, (int(z["n_src"]),), (int(z["n_det"]),), src_high=True)
tol, ns = float(z["tol"]), int(z["n_src"])
op = rd.SchurOperator(g, P.constant_fields(g, z["mu0"]), np.float64, ctx)
res = rd.recycled_cg(op, None, None, z["B"][:, 0], 1e-10, 2 * g.n)
print("plain minres its", res.report.iterations, int(z["minres_its"]), rel(res.correction, z["minres_x"]))
X0, tot = rd.initial_solutions(op, lay, tol)
print("X0", rel(X0, z["X0"]), tot)
gb = rd.GlobalBasis(z["U0"], z["X0"], 0, ctx)
logs = []
for s, mu in enumerate(z["mus"], start=1):
    op.set_fields(P.constant_fields(g, mu))
    pr = rd.process_system(gb, op, lay, tol, s)
    logs.append(np.array([[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in pr.log]))
    print("sys", s, "cols", gb.cols, int(z["cols"][s - 1]), "psi", rel(z["B"][:, ns:].T @ pr.X[:, :ns], z["psi"][s - 1]))
dev = np.concatenate(logs); ref = z["log"]
print("flags equal", np.array_equal(dev[:, [0, 1, 4]], ref[:, [0, 1, 4]]))
d = dev[:, 3] - ref[:, 3]
print("its diff min/max", d.min(), d.max(), "nonzero", np.count_nonzero(d), "of", len(d))
nz = ref[:, 2] > 0
print("init_relres rel diff max", np.abs(dev[nz, 2] / ref[nz, 2] - 1).max())
rec = rd.PerRhsRecycler(z["U0"], z["X0"], ctx)
logs = []
for s, mu in enumerate(z["mus"], start=1):
    op.set_fields(P.constant_fields(g, mu))
    logs.append(np.array([[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in rec.solve_system(op, lay, tol, s).log]))
dev = np.concatenate(logs); ref = z["baseline_log"]
d = dev[:, 3] - ref[:, 3]
print("per-rhs its diff min/max", d.min(), d.max(), "nonzero", np.count_nonzero(d), "of", len(d))
op.set_fields(P.constant_fields(g, z["mus"][1]))
U, K = rd.recycle_space_from_raw(z["rm_W"], z["rm_AW"], ctx)
rhs = z["B"][:, 1]
res = rd.recycled_cg(op, U, K, rhs, 1e-9, 2 * g.n, float(np.linalg.norm(rhs)))
print("recycled its", res.report.iterations, int(z["rm_its"]), rel(res.correction, z["rm_z0"] + z["rm_corr"]))
h = np.asarray(res.report.rel_residual_history); hr = z["rm_hist"]
m = min(len(h), len(hr)); print("hist len", len(h), len(hr), "max rel", np.abs(h[:m] / hr[:m] - 1).max())

# criterion 5
z = np.load(os.path.join(G, "ref_criterion5.npz"))
nx = int(z["cfg"][0]); g = P.GridSpec.reference_2d(nx, nx)
lay = P.make_layout(g, (32,), (32,), src_high=True)
tol, k = float(z["tol"]), int(z["k_eig"])
op = rd.SchurOperator(g, P.constant_fields(g, z["mus"][0]), np.float64, ctx)
gb, X0, lam, U0 = rd.init_basis(op, op, lay, k, tol)
rec = rd.PerRhsRecycler(U0, X0, ctx)
rows = z["rows"]; ours = base = 0
for s in (1, 2):
    op.set_fields(P.constant_fields(g, z["mus"][s]))
    a = rd.process_system(gb, op, lay, tol, s)
    b = rec.solve_system(op, lay, tol, s)
    rr = rows[rows[:, 0] == s]
    da = np.array([r.iterations for r in a.log]) - rr[:, 2]
    db = np.array([r.iterations for r in b.log]) - rr[:, 4]
    print("c5 sys", s, "ours diff", da.min(), da.max(), np.count_nonzero(da), "base diff", db.min(), db.max(), np.count_nonzero(db))
    ir = np.array([r.init_relres for r in a.log]); print("  init_relres max rel", np.abs(ir / rr[:, 3] - 1).max())
    ours += a.inner_iterations; base += b.inner_iterations
print("c5 totals", ours, int(z["ours"]), base, int(z["baseline"]))
