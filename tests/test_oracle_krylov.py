"""Oracle Krylov kernels pinned to the reference's test_krylov.cpp properties
(line numbers cited per test), plus the CG/COCG extension."""
import numpy as np
import pytest

import oracle as orc


def random_spd(n, seed, shift=1.0):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    return M @ M.T / n + shift * np.eye(n)


def rvec(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


@pytest.mark.parametrize("n", [20, 50, 80])
def test_minres_matches_dense(n):  # test_krylov.cpp:42-52
    A = random_spd(n, 100 + n)
    b = rvec(n, 200 + n)
    x, rep = orc.minres(orc.Operator.dense(A), b, 1e-12, 4 * n)
    assert rep.converged
    xr = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
    assert np.linalg.norm(b - A @ x) <= 1e-11 * np.linalg.norm(b)


def test_minres_indefinite():  # :54-62
    A = random_spd(40, 7) - 2.5 * np.eye(40)
    b = rvec(40, 8)
    x, rep = orc.minres(orc.Operator.dense(A), b, 1e-10, 400)
    assert rep.converged
    assert np.linalg.norm(b - A @ x) <= 1e-9 * np.linalg.norm(b)


def test_minres_monotone_and_maxit():  # :64-73
    A = random_spd(60, 11, 0.01)
    x, rep = orc.minres(orc.Operator.dense(A), rvec(60, 12), 1e-14, 5)
    assert not rep.converged and rep.iterations == 5
    assert (np.diff(rep.history) <= 1e-14).all()


def test_recycle_space_invariants():  # :75-85
    A = random_spd(50, 21)
    W = np.stack([rvec(50, 300 + j) for j in range(4)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    U, K = rs.UK()
    assert np.linalg.norm(K.T @ K - np.eye(4)) <= 1e-12
    assert np.linalg.norm(A @ U - K) <= 1e-10 * np.linalg.norm(K)
    assert rs.cols == 4


def test_recycle_space_100_appends():  # :87-102
    n = 120
    A = random_spd(n, 31)
    W = np.stack([rvec(n, 41), rvec(n, 42)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    for t in range(100):
        u = rvec(n, 500 + t)
        rs.append(u, A @ u)
    U, K = rs.UK()
    assert rs.cols == 102
    assert np.linalg.norm(K.T @ K - np.eye(102)) <= 1e-10
    assert np.linalg.norm(A @ U - K) <= 1e-10 * np.linalg.norm(K)


def test_dependent_append_rejected():  # :104-113
    A = random_spd(30, 51)
    W = np.stack([rvec(30, 600 + j) for j in range(3)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    u = W @ np.full(3, 0.7)
    assert not rs.append(u, A @ u)
    assert rs.cols == 3


def test_initial_guess_optimal():  # :115-129
    A = random_spd(40, 61)
    W = np.stack([rvec(40, 700 + j) for j in range(5)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    b = rvec(40, 62)
    z, r = rs.initial_guess(b)
    U, K = rs.UK()
    assert np.linalg.norm(K.T @ r) <= 1e-10 * np.linalg.norm(b)
    assert np.linalg.norm(b - A @ z - r) <= 1e-10 * np.linalg.norm(b)
    c, *_ = np.linalg.lstsq(A @ W, b, rcond=None)
    assert np.linalg.norm(r) <= np.linalg.norm(b - A @ W @ c) + 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("method", [orc.MINRES, orc.CG])
def test_recycled_solve_to_tolerance(method):  # :131-145
    n = 80
    A = random_spd(n, 71, 0.1)
    W = np.stack([rvec(n, 800 + j) for j in range(6)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    b = rvec(n, 72)
    z0, r0 = rs.initial_guess(b)
    res = orc.recycled_solve(method, orc.Operator.dense(A), rs, r0, 1e-10, 4 * n, np.linalg.norm(b))
    assert res.report.converged
    x = z0 + res.correction
    assert np.linalg.norm(b - A @ x) <= 1e-9 * np.linalg.norm(b)
    assert np.linalg.norm(res.image - A @ res.new_direction) <= 1e-12 * np.linalg.norm(res.image)


def _lanczos_opt(A, K, U, r0, m):
    n = A.shape[0]
    P = np.eye(n) - K @ K.T
    V = np.zeros((n, m))
    V[:, 0] = r0 / np.linalg.norm(r0)
    prev = np.zeros(n)
    beta = 0.0
    for j in range(m - 1):
        w = P @ (A @ V[:, j]) - beta * prev
        for _ in range(2):
            w -= V[:, : j + 1] @ (V[:, : j + 1].T @ w)
        beta = np.linalg.norm(w)
        prev = V[:, j].copy()
        V[:, j + 1] = w / beta
    C = np.hstack([U, V])
    AC = A @ C
    c, *_ = np.linalg.lstsq(AC, r0, rcond=None)
    return np.linalg.norm(r0 - AC @ c)


def test_recycled_minres_attains_augmented_ls_optimum():  # :147-184
    n, m = 60, 8
    A = random_spd(n, 81, 0.05)
    W = np.stack([rvec(n, 900 + j) for j in range(4)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    b = rvec(n, 82)
    z0, r0 = rs.initial_guess(b)
    res = orc.recycled_minres(orc.Operator.dense(A), rs, r0, 1e-16, m, np.linalg.norm(b))
    assert res.report.iterations == m
    U, K = rs.UK()
    opt = _lanczos_opt(A, K, U, r0, m)
    got = np.linalg.norm(r0 - A @ res.correction)
    assert got <= opt + 1e-8 * np.linalg.norm(b)


def test_recycled_cg_is_galerkin_over_augmented_space():
    """CG extension: after m steps the correction minimises the A-norm error of
    P A P y = r0 over the Krylov space (Galerkin); the full residual equals the
    projected one."""
    n, m = 60, 8
    A = random_spd(n, 81, 0.05)
    W = np.stack([rvec(n, 900 + j) for j in range(4)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    U, K = rs.UK()
    b = rvec(n, 82)
    z0, r0 = rs.initial_guess(b)
    res = orc.recycled_cg(orc.Operator.dense(A), rs, r0, 1e-16, m, np.linalg.norm(b))
    assert res.report.iterations == m
    P = np.eye(n) - K @ K.T
    PAP = P @ A @ P
    # Krylov basis of PAP from r0
    Kr = np.zeros((n, m))
    v = r0.copy()
    for j in range(m):
        Kr[:, j] = v
        v = PAP @ v
    Q, _ = np.linalg.qr(Kr)
    y_gal = Q @ np.linalg.solve(Q.T @ PAP @ Q, Q.T @ r0)
    assert np.linalg.norm(res.new_direction - y_gal) <= 1e-8 * np.linalg.norm(y_gal)
    # the recurrence residual is the true residual of A g = r0
    assert abs(np.linalg.norm(r0 - A @ res.correction) / np.linalg.norm(b) - res.report.history[-1]) <= 1e-10


@pytest.mark.parametrize("method", [orc.MINRES, orc.CG])
def test_recycling_reduces_iterations(method):  # :186-202
    n = 150
    A = random_spd(n, 91, 0.01)
    b = rvec(n, 92)
    op = orc.Operator.dense(A)
    plain = orc.recycled_solve(method, op, None, b, 1e-8, 4 * n)
    assert plain.report.converged
    w, Vv = np.linalg.eigh(A)
    Wm = Vv[:, :10]
    rs = orc.RecycleSpace(Wm, A @ Wm)
    z0, r0 = rs.initial_guess(b)
    res = orc.recycled_solve(method, op, rs, r0, 1e-8, 4 * n, np.linalg.norm(b))
    assert res.report.converged
    assert res.report.iterations < plain.report.iterations


def test_cg_matches_dense_solve():
    for n in [20, 50, 80]:
        A = random_spd(n, 100 + n)
        b = rvec(n, 200 + n)
        res = orc.recycled_cg(orc.Operator.dense(A), None, b, 1e-12, 4 * n)
        assert res.report.converged
        xr = np.linalg.solve(A, b)
        assert np.linalg.norm(res.correction - xr) <= 1e-8 * np.linalg.norm(xr)


def complex_symmetric(n, seed, shift=1.0, imag=0.3):
    A = random_spd(n, seed, shift)
    return A + 1j * imag * np.diag(np.random.default_rng(seed + 1).uniform(0.5, 1.5, n))


def test_cocg_complex_symmetric_solve_and_bilinear_space():
    n = 60
    A = complex_symmetric(n, 5)
    W = np.stack([rvec(n, 10 + j) + 0j for j in range(5)], 1)
    rs = orc.RecycleSpace(W, A @ W)
    U, K = rs.UK()
    assert np.linalg.norm(K.T @ K - np.eye(5)) <= 1e-12           # bilinear, not Hermitian
    assert np.linalg.norm(A @ U - K) <= 1e-10 * np.linalg.norm(K)
    b = rvec(n, 99) + 0j
    op = orc.Operator.dense(A)
    res = orc.recycled_cg(op, rs, b, 1e-10, 10 * n, np.linalg.norm(b))
    assert res.report.converged
    assert np.linalg.norm(b - A @ res.correction) <= 1e-9 * np.linalg.norm(b)
    plain = orc.recycled_cg(op, None, b, 1e-10, 10 * n)
    assert plain.report.converged
    assert np.linalg.norm(b - A @ plain.correction) <= 1e-9 * np.linalg.norm(b)


def test_eigenpairs_diagonal():  # :204-215
    A = np.diag(np.arange(1.0, 101.0))
    lam, U = orc.smallest_eigenpairs(orc.Operator.dense(A), 3, 1e-10)
    for i in range(3):
        assert lam[i] == pytest.approx(i + 1.0, rel=1e-8)
        assert abs(U[i, i]) == pytest.approx(1.0, rel=1e-6)


def test_eigenpairs_full_spectrum():  # :217-225
    A = random_spd(12, 101)
    lam, U = orc.smallest_eigenpairs(orc.Operator.dense(A), 12, 1e-10)
    ref = np.linalg.eigvalsh(A)
    assert np.allclose(lam, ref, rtol=1e-8)
    assert np.linalg.norm(U.T @ U - np.eye(12)) <= 1e-8


def test_eigenpair_residual_bound():  # :227-237
    A = random_spd(64, 111, 0.2)
    lam, U = orc.smallest_eigenpairs(orc.Operator.dense(A), 6, 1e-8)
    scale = np.abs(A).sum(1).max()
    for i in range(6):
        assert lam[i] > 0
        assert np.linalg.norm(A @ U[:, i] - lam[i] * U[:, i]) <= 1e-8 * scale
    assert (np.diff(lam) >= 0).all()


def test_thin_qr_and_qrcp_known_rank():
    rng = np.random.default_rng(3)
    n = 600
    for m, want in [(64, 64), (256, 219)]:
        Q, _ = np.linalg.qr(rng.standard_normal((n, m)))
        A = Q * (0.9 ** np.arange(m))
        A = A[:, rng.permutation(m)]
        rank, perm, rdiag, Qk = orc.qrcp(A, 1e-10, normalize=False)
        assert rank == want
        assert np.linalg.norm(Qk.T @ Qk - np.eye(rank)) <= 1e-12
    M = rng.standard_normal((50, 7)) + 1j * rng.standard_normal((50, 7))
    Q, R = orc.thin_qr(M)
    assert np.linalg.norm(Q @ R - M) <= 1e-13 * np.linalg.norm(M)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(7)) <= 1e-13
