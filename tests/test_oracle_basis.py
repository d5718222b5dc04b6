"""Oracle basis builder (Algorithm 2) pinned to the reference's
test_basis.cpp and acceptance.cpp properties (line numbers per test)."""
import numpy as np
import pytest

import oracle as orc
from helpers import Desk, fom_transfer, rom_transfer
from paper_1602_00138_b200 import problem as P


def init(desk, offset, k, tol, method=orc.CG, dtype=np.float64):
    op = desk.op(offset, dtype)
    op_r = desk.op(offset)
    gb, X0, lam, U0 = orc.init_basis(op, op_r, desk.layout, k, tol, method)
    return gb


def rvec(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


@pytest.mark.parametrize("method", [orc.MINRES, orc.CG])
def test_blockwise_image_qr(method):  # test_basis.cpp:65-83
    d = Desk(15, 3, 3)
    gb = init(d, 0.0, 4, 1e-8, method)
    gb.refresh(d.op(0.0))
    r = gb.cols
    Kf = d.A(0.0) @ gb.V
    K, R = gb.K_img, gb.R
    assert np.linalg.norm(K @ R - Kf) <= 1e-12 * np.linalg.norm(Kf)
    assert np.linalg.norm(K.T @ K - np.eye(r)) <= 1e-12
    assert np.all(np.tril(R, -1) == 0.0)
    Q, _ = np.linalg.qr(Kf)
    assert np.allclose(np.abs(np.diag(Q.T @ K)), 1.0, atol=1e-10)


def test_append_consistent_with_refresh():  # :85-108
    d = Desk(15, 3, 3)
    gb = init(d, 0.0, 4, 1e-8)
    op = d.op(0.0)
    gb.refresh(op)
    A = d.A(0.0)
    for t in range(5):
        y = rvec(d.grid.n, 40 + t)
        assert gb.append(y, A @ y)
    r = gb.cols
    Kf = A @ gb.V
    assert np.linalg.norm(gb.K_img @ gb.R - Kf) <= 1e-10 * np.linalg.norm(Kf)
    assert np.linalg.norm(gb.K_img.T @ gb.K_img - np.eye(r)) <= 1e-10
    b = rvec(d.grid.n, 99)
    xi = gb.solve_projected(b)
    gb.refresh(op)
    xr = gb.solve_projected(b)
    assert np.linalg.norm(xi - xr) <= 1e-9 * np.linalg.norm(xr)


def test_dependent_append_dropped():  # :110-121
    d = Desk(15, 3, 3)
    gb = init(d, 0.0, 4, 1e-8)
    gb.refresh(d.op(0.0))
    before = gb.cols
    y = gb.V @ np.full(before, 0.3)
    assert not gb.append(y, d.A(0.0) @ y)
    assert gb.cols == before


def test_projected_solve_is_ls():  # :123-136
    d = Desk(15, 3, 3)
    gb = init(d, 0.0, 4, 1e-8)
    gb.refresh(d.op(0.0))
    b = rvec(d.grid.n, 7)
    x = gb.solve_projected(b)
    AV = d.A(0.0) @ gb.V
    c, *_ = np.linalg.lstsq(AV, b, rcond=None)
    assert np.linalg.norm(x - gb.V @ c) <= 1e-8 * np.linalg.norm(x)


@pytest.mark.parametrize("method", [orc.MINRES, orc.CG])
def test_reprocessing_covered_system_zero_iterations(method):  # :138-148
    d = Desk(21, 4, 4)
    gb = init(d, 0.0, 6, 1e-7, method)
    pr = orc.process_system(gb, d.op(0.0), d.layout, 1e-7, 1, method=method)
    assert all(r.iterations == 0 and not r.appended for r in pr.log)
    assert pr.appends == 0


@pytest.mark.parametrize("method", [orc.MINRES, orc.CG])
def test_growth_accounting_and_residuals(method):  # :150-193, acceptance C4 :276-313
    d = Desk(21, 4, 4)
    k_eig, n_rhs = 6, 8
    gb = init(d, 0.0, k_eig, 1e-7, method)
    assert gb.cols == k_eig + n_rhs and gb.eig_block == k_eig
    appends, rows, totals = 0, [], []
    for sys in (1, 2):
        pr = orc.process_system(gb, d.op(0.02 * sys), d.layout, 1e-7, sys, method=method)
        appends += pr.appends
        rows += pr.log
        totals.append(pr.inner_iterations)
        A = d.A(0.02 * sys)
        for j in range(n_rhs):
            b = d.B[:, j]
            assert np.linalg.norm(b - A @ pr.X[:, j]) <= 1e-7 * np.linalg.norm(b)
    assert gb.cols == k_eig + n_rhs + appends
    assert sum(r.appended for r in rows) == appends
    assert (gb.markers == 2).sum() == appends
    assert totals[1] < totals[0]


def test_per_rhs_space_layout():  # :195-208
    d = Desk(21, 4, 4)
    gb = init(d, 0.0, 6, 1e-7)
    orc.process_system(gb, d.op(0.02), d.layout, 1e-7, 1)
    r = gb.cols
    for j in range(8):
        cols = gb.space(j)
        assert cols[:6] == list(range(6))
        assert cols[6] == 6 + j
        assert all(c < r for c in cols)


def test_bitwise_determinism():  # :210-223
    def build():
        d = Desk(21, 4, 4)
        gb = init(d, 0.0, 6, 1e-7)
        orc.process_system(gb, d.op(0.02), d.layout, 1e-7, 1)
        return gb.V
    V1, V2 = build(), build()
    assert V1.shape == V2.shape and V1.tobytes() == V2.tobytes()


@pytest.mark.parametrize("cfg", ["T2", "T2c", "T3", "T3c"])
def test_baseline_configs_build_and_residuals(cfg):
    """BASELINE-shaped extension (variable D, 3D, complex shift, COCG, cap):
    every solution passes the explicit residual check (test_basis.cpp:180-193)."""
    c = P.CONFIGS[cfg]
    g = c.grid
    lay = c.layout()
    f0 = c.fields(0)
    op0 = orc.Operator.grid(g, f0, c.dtype)
    op0r = orc.Operator.grid(g, f0)
    gb, X0, lam, U0 = orc.init_basis(op0, op0r, lay, c.k, c.tol, cap=c.cap)
    B = lay.dense(g.n)
    zero_rows, totals = 0, []
    for s, (pt, w) in enumerate(c.systems(), start=1):
        f = c.fields(pt, w)
        op = orc.Operator.grid(g, f, c.dtype)
        pr = orc.process_system(gb, op, lay, c.tol, s)
        A = op.matrix() if g.n <= 2000 else None
        if A is not None:
            for j in range(lay.n_rhs):
                assert np.linalg.norm(B[:, j] - A @ pr.X[:, j]) <= c.tol * np.linalg.norm(B[:, j])
        zero_rows += sum(r.iterations == 0 for r in pr.log)
        totals.append(pr.inner_iterations)
        if c.cap:
            assert gb.cols <= c.cap
    assert gb.cols >= c.k + lay.n_rhs


def test_svd_and_rrqr_compressed_rom_match_algorithm2():  # acceptance C7 :362-400
    d = Desk(21, 4, 4)
    offs = [0.0, 0.02, 0.04, 0.06]
    gb = init(d, offs[0], 6, 1e-7)
    S = [gb.V.copy()]   # U0, X0
    for s, o in enumerate(offs[1:], start=1):
        pr = orc.process_system(gb, d.op(o), d.layout, 1e-7, s)
        S.append(pr.X)
    S = np.hstack(S)
    U, sv, _ = np.linalg.svd(S, full_matrices=False)
    rank = int((sv > 1e-10 * sv[0]).sum())
    V_svd = U[:, :rank]
    V_qr = gb.V
    rk, perm, rdiag, Q = orc.qrcp(V_qr, 1e-10)
    Bt, Ct = d.B[:, :4], d.B[:, 4:]
    worst = worst_rr = 0.0
    for o in offs:
        A = d.A(o)
        a = rom_transfer(V_qr, A, Bt, Ct)
        b = rom_transfer(V_svd, A, Bt, Ct)
        c = rom_transfer(Q, A, Bt, Ct)
        worst = max(worst, np.linalg.norm(a - b) / np.linalg.norm(a))
        worst_rr = max(worst_rr, np.linalg.norm(a - c) / np.linalg.norm(a))
        # ROM at basis parameters vs FOM (criterion 3)
        psi = fom_transfer(A, Bt, Ct)
        assert np.linalg.norm(a - psi) / np.linalg.norm(psi) <= 1e-5
    assert worst <= 1e-4 and worst_rr <= 1e-4


@pytest.mark.parametrize("method", [orc.MINRES, orc.CG])
def test_baseline_recycler_per_rhs_growth_only(method):  # test_basis.cpp:225-240
    d = Desk(21, 4, 4)
    k = 6
    gb, X0, lam, U0 = orc.init_basis(d.op(0.0), d.op(0.0), d.layout, k, 1e-7, method)
    base = orc.PerRhsRecycler(U0, X0)
    for s in (1, 2):
        pr = base.solve_system(d.op(0.02 * s), d.layout, 1e-7, s, method=method)
        A = d.A(0.02 * s)
        res = np.linalg.norm(d.B - A @ pr.X, axis=0) / np.linalg.norm(d.B, axis=0)
        assert res.max() <= 1e-7
        # appends only where the RHS iterated; no cross-RHS sharing (basis.cpp:252-258)
        assert pr.appends == sum(r.appended for r in pr.log)
        assert all(r.appended == (r.iterations > 0) for r in pr.log)
