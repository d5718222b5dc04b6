"""The CUDA path against THE REFERENCE'S OWN OUTPUT (tests/golden/ref_*.npz,
produced by scripts/make_ref_golden.py from the reference's sources compiled
unmodified; see tests/test_ref_golden.py).  Reads only the committed fixtures:
nothing from /root/reference or oracle/ is needed on the GPU box.

Every test runs twice (fixture `ctx`):

* `minres` -- the context's inner solver switched to the reference's own
  recycled MINRES on the device (rd_ctx_set_solver 1; krylov.cpp:17-98,
  147-179).  Same algorithm as the reference, so the bars are the reference's
  numbers themselves: IDENTICAL iteration count and append flag on every
  BuildLog row, init_relres within 1e-5 relative, solutions and transfer
  functions within 1e-10, criterion 5 totals exactly 4177 / 9403.
* `cg` -- the product default (BASELINE asks for CG on SPD systems) on the
  same deflated operator to the same explicit-residual tolerance: identical
  append flags, iterations within [-1, +3] of the reference's MINRES counts
  (CG's residual is not the minimal one, it needs 0..2 more), init_relres
  within 5e-3 relative, solutions / transfer functions within 1e-6.
"""
import os

import numpy as np
import pytest

from paper_1602_00138_b200 import problem as P

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def rd():
    from paper_1602_00138_b200 import build, romdot
    build.build()
    return romdot


def load(name):
    return np.load(os.path.join(HERE, name))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def log_array(rows):
    return np.array([[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in rows])


@pytest.fixture(params=["minres", "cg"])
def ctx(rd, request):
    c = rd.Context(0)
    c.set_solver(rd.Context.MINRES if request.param == "minres" else rd.Context.CG)
    c.exact = request.param == "minres"
    return c


def check_rows(dev, refrows, what, exact):
    assert np.array_equal(dev[:, [0, 1, 4]], refrows[:, [0, 1, 4]]), what  # system, rhs, appended
    diff = dev[:, 3] - refrows[:, 3]
    if exact:
        assert not diff.any(), (what, diff.min(), diff.max())
    else:
        assert diff.min() >= -1 and diff.max() <= 3, (what, diff.min(), diff.max())
    assert np.array_equal(dev[:, 3] == 0, refrows[:, 3] == 0), what  # the same rows are served by the basis
    assert np.allclose(dev[:, 2], refrows[:, 2], rtol=1e-5 if exact else 5e-3), what


def desk(z):
    n = int(z["n"])
    g = P.GridSpec.reference_2d(n, n)
    return g, P.make_layout(g, (int(z["n_src"]),), (int(z["n_det"]),), src_high=True)


def supports(dmu):
    out = []
    for col in dmu.T:
        ix = np.nonzero(col)[0]
        out.append((ix, col[ix]))
    return out


def test_operator_and_seed_match_reference(rd, ctx):  # grid.cpp:95-97, krylov.cpp:181-280, basis.cpp:136-155
    z = load("ref_desk.npz")
    g, lay = desk(z)
    op = rd.SchurOperator(g, P.constant_fields(g, z["mu0"]), np.float64, ctx)
    y = op.apply(z["apply_x"])
    assert np.abs(y - z["apply_y"]).max() <= 1e-14 * np.abs(z["apply_y"]).max()
    lam, U0 = rd.smallest_eigenpairs(op, int(z["k"]), 1e-8)
    assert np.allclose(lam, z["eigenvalues"], rtol=1e-8)
    assert np.linalg.svd(U0.T @ z["U0"], compute_uv=False).min() >= 1 - 1e-8
    X0, _ = rd.initial_solutions(op, lay, float(z["tol"]))
    assert rel(X0, z["X0"]) <= (1e-12 if ctx.exact else 1e-6)
    # plain (undeflated) solve against the reference's MINRES solution (krylov.cpp:100-104)
    res = rd.recycled_cg(op, None, None, z["B"][:, 0], 1e-10, 2 * g.n)
    assert rel(res.correction, z["minres_x"]) <= (1e-12 if ctx.exact else 1e-8)
    assert abs(res.report.iterations - int(z["minres_its"])) <= (0 if ctx.exact else 3)


def test_process_system_matches_reference_buildlog(rd, ctx):  # basis.cpp:157-207
    z = load("ref_desk.npz")
    g, lay = desk(z)
    tol, ns = float(z["tol"]), int(z["n_src"])
    xt = 1e-10 if ctx.exact else 1e-6
    gb = rd.GlobalBasis(z["U0"], z["X0"], 0, ctx)
    op = rd.SchurOperator(g, P.constant_fields(g, z["mus"][0]), np.float64, ctx)
    Ct = z["B"][:, ns:]
    logs = []
    for s, mu in enumerate(z["mus"], start=1):
        op.set_fields(P.constant_fields(g, mu))
        pr = rd.process_system(gb, op, lay, tol, s)
        logs.append(log_array(pr.log))
        assert gb.cols == int(z["cols"][s - 1])
        assert rel(Ct.T @ pr.X[:, :ns], z["psi"][s - 1]) <= xt
        assert np.allclose(np.linalg.norm(pr.X, axis=0), z["xnorm"][s - 1], rtol=xt)
    check_rows(np.concatenate(logs), z["log"], "global basis", ctx.exact)
    assert np.array_equal(gb.markers, z["markers"])
    assert [len(gb.space(j)) for j in range(lay.n_rhs)] == z["spaces"].tolist()
    # reduced model on the device-built basis at a new parameter vs the reference's ReducedModel on its basis
    op.set_fields(P.constant_fields(g, z["rom_mu"]))
    rom = rd.ReducedModel(gb.V, None, ctx)
    assert rel(rom.transfer(op, lay), z["rom_psi"]) <= (1e-9 if ctx.exact else 1e-6)
    J = rom.jacobian(op, lay, supports(z["pals_jac_cols"]), -g.h ** 2)
    assert rel(J, z["rom_jac"]) <= (1e-8 if ctx.exact else 1e-5)
    # full-order transfer / Jacobian (rom.cpp:71-129) vs the reference's direct solves
    assert rel(rd.fom_transfer(op, lay, 1e-12)[0], z["fom_psi"]) <= 1e-8
    assert rel(rd.fom_jacobian(op, lay, supports(z["pals_jac_cols"]), -g.h ** 2, 1e-12), z["fom_jac"]) <= 1e-7


def test_per_rhs_recycler_matches_reference(rd, ctx):  # basis.cpp:209-266
    z = load("ref_desk.npz")
    g, lay = desk(z)
    rec = rd.PerRhsRecycler(z["U0"], z["X0"], ctx)
    op = rd.SchurOperator(g, P.constant_fields(g, z["mus"][0]), np.float64, ctx)
    logs = []
    for s, mu in enumerate(z["mus"], start=1):
        op.set_fields(P.constant_fields(g, mu))
        logs.append(log_array(rec.solve_system(op, lay, float(z["tol"]), s).log))
    check_rows(np.concatenate(logs), z["baseline_log"], "per-RHS only", ctx.exact)


def test_recycled_solve_matches_reference(rd, ctx):  # krylov.cpp:106-115, 147-179
    z = load("ref_desk.npz")
    g, lay = desk(z)
    op = rd.SchurOperator(g, P.constant_fields(g, z["mus"][1]), np.float64, ctx)
    U, K = rd.recycle_space_from_raw(z["rm_W"], z["rm_AW"], ctx)
    rhs = z["B"][:, 1]
    res = rd.recycled_cg(op, U, K, rhs, 1e-9, 2 * g.n, float(np.linalg.norm(rhs)))
    if ctx.exact:  # the reference's residual history, step by step
        assert res.report.iterations == int(z["rm_its"])
        assert np.allclose(res.report.rel_residual_history, z["rm_hist"], rtol=1e-9, atol=0)
        assert rel(res.correction, z["rm_z0"] + z["rm_corr"]) <= 1e-12
    assert -1 <= res.report.iterations - int(z["rm_its"]) <= 3
    # the reference returns g for the projected right-hand side and leaves z0 = U K^T rhs
    # (initial_guess) to the caller; the device entry point returns z0 + g (K^T rhs = 0 in every
    # call the reference's builder makes, where the two coincide)
    assert rel(res.correction, z["rm_z0"] + z["rm_corr"]) <= 1e-6
    assert rel(U @ (K.T @ rhs), z["rm_z0"]) <= 1e-10


def test_criterion5_on_the_reference_phantom(rd, ctx):  # acceptance.cpp:314-334, harness.cpp:208-251
    """The reference's acceptance criterion 5 on its own PaLS phantom (121^2,
    32 + 32, seed 1234, tol 1e-7), run on the device from the DEVICE's own seed
    (device Lanczos eigenvectors + device X0 solves).

    minres: every one of the 2 x 64 BuildLog rows of both arms has the
    reference's iteration count, the totals are the reference's 4177 / 9403 and
    `ours * 2 <= baseline` (acceptance.cpp:325) holds.
    cg: same rows served by the basis; CG stops on the same explicit-residual
    bound but its residual is not the minimal one, which at this loose tolerance
    costs 10..16 iterations per per-RHS-only solve (measured: 5406 / 11046); the
    reference's bar `ours * 2 <= baseline` still holds."""
    z = load("ref_criterion5.npz")
    nx = int(z["cfg"][0])
    g = P.GridSpec.reference_2d(nx, nx)
    lay = P.make_layout(g, (32,), (32,), src_high=True)
    tol, k = float(z["tol"]), int(z["k_eig"])
    op = rd.SchurOperator(g, P.constant_fields(g, z["mus"][0]), np.float64, ctx)
    gb, X0, lam, U0 = rd.init_basis(op, op, lay, k, tol)
    rec = rd.PerRhsRecycler(U0, X0, ctx)
    rows = z["rows"]
    ours = base = 0
    for s in (1, 2):
        op.set_fields(P.constant_fields(g, z["mus"][s]))
        a = rd.process_system(gb, op, lay, tol, s)
        b = rec.solve_system(op, lay, tol, s)
        rr = rows[rows[:, 0] == s]
        ia = np.array([r.iterations for r in a.log])
        ib = np.array([r.iterations for r in b.log])
        if ctx.exact:
            assert np.array_equal(ia, rr[:, 2]) and np.array_equal(ib, rr[:, 4]), s
            assert np.allclose([r.init_relres for r in a.log], rr[:, 3], rtol=1e-4)
        else:
            assert (ib - rr[:, 4]).min() >= -2 and (ib - rr[:, 4]).max() <= 20, s
            # which rows the basis serves with 0 iterations depends on the corrections appended
            # before them (one near-tolerance row flips under CG): only the count is compared
            assert abs(int((ia == 0).sum()) - int((rr[:, 2] == 0).sum())) <= 2, s
        ours += a.inner_iterations
        base += b.inner_iterations
    if ctx.exact:
        assert (ours, base) == (int(z["ours"]), int(z["baseline"])), (ours, base)
    else:
        assert ours <= 1.35 * int(z["ours"]) and base <= 1.25 * int(z["baseline"]), (ours, base)
    assert ours * 2 <= base


def test_hybrid_sequence_matches_reference(rd, ctx):  # inversion.cpp:53-106
    """The reference's HybridEvaluator run: K_* = 3 systems through the device
    builder from the reference's seed, then the device reduced model on V."""
    z = load("ref_hybrid.npz")
    nx = int(z["cfg"][0])
    g = P.GridSpec.reference_2d(nx, nx)
    ns = 6
    lay = P.make_layout(g, (ns,), (ns,), src_high=True)
    tol = 1e-8
    xt = 1e-9 if ctx.exact else 1e-6
    gb = rd.GlobalBasis(z["U0"], z["X0"], 0, ctx)
    op = rd.SchurOperator(g, P.constant_fields(g, z["mus"][0]), np.float64, ctx)
    Ct = z["B"][:, ns:]
    logs = []
    for s in (1, 2, 3):
        op.set_fields(P.constant_fields(g, z["mus"][s]))
        pr = rd.process_system(gb, op, lay, tol, s)
        logs.append(log_array(pr.log))
        assert rel(Ct.T @ pr.X[:, :ns], z[f"psi{s}"]) <= xt
        if s == 1:
            Xs, Zd = pr.X[:, :ns], pr.X[:, ns:]
            J = np.stack([-float(z["h2"]) * ((Zd * dk[:, None]).T @ Xs).ravel(order="F") for dk in z["dmu1"].T], axis=1)
            assert rel(J, z["jac1"]) <= 10 * xt
    check_rows(np.concatenate(logs), z["log"], "hybrid build", ctx.exact)
    assert gb.cols == int(z["state3"][0])
    op.set_fields(P.constant_fields(g, z["mus"][4]))
    rom = rd.ReducedModel(gb.V, None, ctx)
    assert rel(rom.transfer(op, lay), z["psi4_rom"]) <= xt
    assert rel(rom.jacobian(op, lay, supports(z["dmu4"]), -float(z["h2"])), z["jac4_rom"]) <= 10 * xt
