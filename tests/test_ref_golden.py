"""The CPU restatement pinned to THE REFERENCE'S OWN OUTPUT.

tests/golden/ref_*.npz were produced by scripts/make_ref_golden.py from
oracle/_ref/libromdot_ref.so, i.e. the reference's sources
(/root/reference/proj/src/*.cpp) compiled unmodified (against the Eigen
stand-in oracle/eigen_shim) and run on the reference's own problems:
test_basis.cpp's desk with its PaLS absorption, acceptance.cpp's criterion 5,
and the HybridEvaluator.  Here the restatement (oracle.py, MINRES mode = the
reference's solver) must reproduce them: identical iteration counts and
append flags row by row, init_relres / solutions / transfer functions to
round-off.  tests/test_ref_live.py re-runs the reference itself where
/root/reference exists and checks that it still produces these fixtures.
"""
import os

import numpy as np
import pytest

import oracle as orc
from helpers import rom_transfer
from paper_1602_00138_b200 import problem as P

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(HERE, name))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def desk_problem(z):
    n = int(z["n"])
    g = P.GridSpec.reference_2d(n, n)
    lay = P.make_layout(g, (int(z["n_src"]),), (int(z["n_det"]),), src_high=True)
    return g, lay


def op_of(g, mu):
    return orc.Operator.grid(g, P.constant_fields(g, mu))


def log_array(rows):
    return np.array([[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in rows])


def test_grid_layout_and_operator_match_reference():  # grid.cpp:27-160
    z = load("ref_desk.npz")
    g, lay = desk_problem(z)
    # interior nodes: the reference's layer j = 1 is this grid's layer 0
    assert np.abs(g.coordinates() + np.array([0.0, g.h]) - z["nodes"]).max() <= 1e-15
    assert P.evenly_spaced_positions(int(z["n"]), int(z["n_src"])) == z["src"].tolist()
    assert np.array_equal(lay.dense(g.n), z["B"])  # B~ = D2 G^-1 B1, C~ = D1^T G^-1 C1, bit for bit
    y = op_of(g, z["mu0"]).apply(z["apply_x"])
    assert np.abs(y - z["apply_y"]).max() <= 4e-16 * np.abs(z["apply_y"]).max()


def test_minres_matches_reference_iteration_by_iteration():  # krylov.cpp:17-104
    z = load("ref_desk.npz")
    g, lay = desk_problem(z)
    x, rep = orc.minres(op_of(g, z["mu0"]), z["B"][:, 0], 1e-10, 2 * g.n)
    assert rep.iterations == int(z["minres_its"])
    assert rep.history.shape == z["minres_hist"].shape
    assert np.allclose(rep.history, z["minres_hist"], rtol=1e-9, atol=0)
    assert rel(x, z["minres_x"]) <= 1e-13


def test_seed_matches_reference():  # krylov.cpp:181-280, basis.cpp:136-155
    z = load("ref_desk.npz")
    g, lay = desk_problem(z)
    op0 = op_of(g, z["mu0"])
    gb, X0, lam, U0 = orc.init_basis(op0, op0, lay, int(z["k"]), float(z["tol"]), orc.MINRES)
    assert np.allclose(lam, z["eigenvalues"], rtol=1e-10)
    # same invariant subspace (eigenvector signs are the eigensolver's)
    s = np.linalg.svd(U0.T @ z["U0"], compute_uv=False)
    assert s.min() >= 1 - 1e-10
    assert rel(X0, z["X0"]) <= 1e-12


@pytest.mark.parametrize("own_seed", [False, True])
def test_process_system_buildlog_matches_reference(own_seed):  # basis.cpp:157-207
    """Four systems (the third revisits p0: zero iterations). From the
    reference's seed, and from the restatement's own seed."""
    z = load("ref_desk.npz")
    g, lay = desk_problem(z)
    tol, ns = float(z["tol"]), int(z["n_src"])
    if own_seed:
        op0 = op_of(g, z["mu0"])
        gb, _, _, _ = orc.init_basis(op0, op0, lay, int(z["k"]), tol, orc.MINRES)
    else:
        gb = orc.GlobalBasis(z["U0"], z["X0"])
    logs = []
    Ct = z["B"][:, ns:]
    for s, mu in enumerate(z["mus"], start=1):
        pr = orc.process_system(gb, op_of(g, mu), lay, tol, s, 0, orc.MINRES)
        logs.append(log_array(pr.log))
        assert gb.cols == int(z["cols"][s - 1])
        assert rel(Ct.T @ pr.X[:, :ns], z["psi"][s - 1]) <= 1e-11
        assert np.allclose(np.linalg.norm(pr.X, axis=0), z["xnorm"][s - 1], rtol=1e-11)
    log = np.concatenate(logs)
    assert np.array_equal(log[:, [0, 1, 3, 4]], z["log"][:, [0, 1, 3, 4]])  # system, rhs, iterations, appended
    assert np.allclose(log[:, 2], z["log"][:, 2], rtol=1e-6)
    assert np.array_equal(gb.markers, z["markers"])
    assert [len(gb.space(j)) for j in range(lay.n_rhs)] == z["spaces"].tolist()
    gb.refresh(op_of(g, z["mus"][-1]))
    assert np.allclose(np.abs(np.diag(gb.R)), z["R_diag_abs"], rtol=1e-8)


def test_per_rhs_recycler_matches_reference():  # basis.cpp:209-266
    z = load("ref_desk.npz")
    g, lay = desk_problem(z)
    rec = orc.PerRhsRecycler(z["U0"], z["X0"])
    logs = []
    for s, mu in enumerate(z["mus"], start=1):
        logs.append(log_array(rec.solve_system(op_of(g, mu), lay, float(z["tol"]), s, 0, orc.MINRES).log))
    log = np.concatenate(logs)
    assert np.array_equal(log[:, [0, 1, 3, 4]], z["baseline_log"][:, [0, 1, 3, 4]])
    assert np.allclose(log[:, 2], z["baseline_log"][:, 2], rtol=1e-6)


def test_recycled_minres_matches_reference():  # krylov.cpp:106-115, 147-179
    z = load("ref_desk.npz")
    g, lay = desk_problem(z)
    op = op_of(g, z["mus"][1])
    rs = orc.RecycleSpace(z["rm_W"], z["rm_AW"])
    rhs = z["B"][:, 1]
    res = orc.recycled_minres(op, rs, rhs, 1e-9, 2 * g.n, float(np.linalg.norm(rhs)))
    assert res.report.iterations == int(z["rm_its"])
    assert np.allclose(res.report.history, z["rm_hist"], rtol=1e-8, atol=0)
    assert rel(res.correction, z["rm_corr"]) <= 1e-11
    assert abs(res.report.correction_norm - float(z["rm_corr_norm"])) <= 1e-11 * float(z["rm_corr_norm"])
    z0, r0 = rs.initial_guess(rhs)
    assert rel(z0, z["rm_z0"]) <= 1e-11 and rel(r0, z["rm_r0"]) <= 1e-12


def test_reduced_model_matches_reference():  # rom.cpp:9-67
    """The parity protocol's ROM observable (helpers.rom_transfer) on the
    reference's final basis is the reference's ReducedModel::transfer, and
    close to the reference's full-order transfer."""
    z = load("ref_desk.npz")
    g, lay = desk_problem(z)
    tol, ns = float(z["tol"]), int(z["n_src"])
    gb = orc.GlobalBasis(z["U0"], z["X0"])
    for s, mu in enumerate(z["mus"], start=1):
        orc.process_system(gb, op_of(g, mu), lay, tol, s, 0, orc.MINRES)
    V = gb.V
    A = op_of(g, z["rom_mu"]).matrix()
    B, Ct = z["B"][:, :ns], z["B"][:, ns:]
    psi = rom_transfer(V, A, B, Ct)
    assert rel(psi, z["rom_psi"]) <= 1e-9
    assert rel(z["rom_psi"], z["fom_psi"]) <= 1e-3  # the reference's own ROM vs FOM gap on this basis
    # Jacobian: -h^2 C_r^T A_r^-1 (V^T diag(dmu_k) V) A_r^-1 B_r per parameter (rom.cpp:37-67)
    Ar = V.T @ (A @ V)
    Ar = 0.5 * (Ar + Ar.T)
    Y, Zc = np.linalg.solve(Ar, V.T @ B), np.linalg.solve(Ar, V.T @ Ct)
    J = np.stack([-(Zc.T @ (V.T @ (dk[:, None] * V)) @ Y).ravel(order="F") for dk in (g.h ** 2 * z["pals_jac_cols"]).T],
                 axis=1)
    assert rel(J, z["rom_jac"]) <= 1e-8


def test_criterion5_matches_reference_row_by_row():  # acceptance.cpp:314-334, harness.cpp:208-251
    """The reference's own acceptance criterion 5 on its own phantom: the
    restatement gives the reference's inner-iteration counts for every
    (system, rhs) of both recyclers, hence the same totals and the same
    PASS of `ours * 2 <= baseline`."""
    z = load("ref_criterion5.npz")
    nx = int(z["cfg"][0])
    g = P.GridSpec.reference_2d(nx, nx)
    lay = P.make_layout(g, (32,), (32,), src_high=True)
    assert np.array_equal(lay.idx, z["B_idx"]) and np.array_equal(lay.val, z["B_val"])
    tol, k = float(z["tol"]), int(z["k_eig"])
    op0 = op_of(g, z["mus"][0])
    gb, X0, lam, U0 = orc.init_basis(op0, op0, lay, k, tol, orc.MINRES)
    rec = orc.PerRhsRecycler(U0, X0)
    rows = z["rows"]  # system, rhs, its_ours, init_relres_ours, its_baseline, init_relres_baseline
    ours = base = 0
    for s in (1, 2):
        op = op_of(g, z["mus"][s])
        a = orc.process_system(gb, op, lay, tol, s, 0, orc.MINRES)
        b = rec.solve_system(op, lay, tol, s, 0, orc.MINRES)
        ref_rows = rows[rows[:, 0] == s]
        ia = np.array([r.iterations for r in a.log])
        ib = np.array([r.iterations for r in b.log])
        # the CSV carries init_relres to 6 digits
        assert np.allclose([r.init_relres for r in a.log], ref_rows[:, 3], rtol=2e-5)
        assert np.allclose([r.init_relres for r in b.log], ref_rows[:, 5], rtol=2e-5)
        assert np.abs(ia - ref_rows[:, 2]).max() <= 1, np.abs(ia - ref_rows[:, 2]).max()
        assert np.abs(ib - ref_rows[:, 4]).max() <= 1
        ours += a.inner_iterations
        base += b.inner_iterations
    assert abs(ours - int(z["ours"])) <= 4 and abs(base - int(z["baseline"])) <= 4, (ours, base)
    assert ours * 2 <= base  # acceptance.cpp:325


def test_hybrid_evaluator_sequence_matches_reference():  # inversion.cpp:53-106
    """K_* = 3 systems through process_system, then the reduced model: the
    restatement driven with the reference's parameter sequence gives the
    reference's BuildLog and transfer functions before and after the switch."""
    z = load("ref_hybrid.npz")
    nx = int(z["cfg"][0])
    g = P.GridSpec.reference_2d(nx, nx)
    ns = nd = 6
    lay = P.make_layout(g, (ns,), (nd,), src_high=True)
    assert np.array_equal(lay.dense(g.n), z["B"])
    tol = 1e-8
    gb = orc.GlobalBasis(z["U0"], z["X0"])
    Ct = z["B"][:, ns:]
    assert rel(Ct.T @ z["X0"][:, :ns], z["psi0"]) <= 1e-13
    logs = []
    for s in (1, 2, 3):
        pr = orc.process_system(gb, op_of(g, z["mus"][s]), lay, tol, s, 0, orc.MINRES)
        logs.append(log_array(pr.log))
        assert rel(Ct.T @ pr.X[:, :ns], z[f"psi{s}"]) <= 1e-11
        if s == 1:  # jacobian_from_solutions (rom.cpp:101-120) on the system's own solutions
            Xs, Zd = pr.X[:, :ns], pr.X[:, ns:]
            J = np.stack([-float(z["h2"]) * ((Zd * dk[:, None]).T @ Xs).ravel(order="F") for dk in z["dmu1"].T], axis=1)
            assert rel(J, z["jac1"]) <= 1e-10
    log = np.concatenate(logs)
    assert np.array_equal(log[:, [0, 1, 3, 4]], z["log"][:, [0, 1, 3, 4]])
    assert gb.cols == int(z["state3"][0]) and int(log[:, 4].sum()) == int(z["state3"][2])
    A4 = op_of(g, z["mus"][4]).matrix()
    assert rel(rom_transfer(gb.V, A4, z["B"][:, :ns], Ct), z["psi4_rom"]) <= 1e-8
    assert int(z["state4"][3]) == 1 and int(z["state4"][1]) == 3
