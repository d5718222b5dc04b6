"""The restatement against THE REFERENCE ITSELF, run live.

oracle/_ref/libromdot_ref.so is /root/reference/proj/src/*.cpp compiled
unmodified (oracle/Makefile target _ref; Eigen stand-in: oracle/eigen_shim).
These tests call the reference's functions and the restatement's on the same
inputs; they run wherever the library can be built or was shipped, and skip
otherwise (the committed fixtures of tests/test_ref_golden.py still pin the
restatement there).  The first test closes the loop: the reference, re-run,
reproduces the committed fixtures.
"""
import os

import numpy as np
import pytest

import oracle as orc
import ref
from paper_1602_00138_b200 import problem as P

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built and /root/reference absent")

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def desk_params(offset):  # Desk::params, test_basis.cpp:43-52
    p = np.zeros(16)
    for j in range(4):
        p[j] = 0.6 + offset
        p[4 + j] = 0.9
        p[8 + 2 * j] = 1.0 + 2.0 * (j % 2)
        p[8 + 2 * j + 1] = 1.0 + 2.0 * (j // 2)
    return p


class Desk:
    """test_basis.cpp:16-53 on both sides: reference grid + PaLS, restatement GridSpec."""

    def __init__(self, n, ns, nd):
        self.rg = ref.Grid(n, n)
        self.nodes = self.rg.interior_nodes()
        self.pals = ref.Pals(m_bumps=4)
        self.B = self.rg.layout(ref.evenly_spaced_positions(n, ns), ref.evenly_spaced_positions(n, nd))
        self.g = P.GridSpec.reference_2d(n, n)
        self.lay = P.make_layout(self.g, (ns,), (nd,), src_high=True)
        self.ns, self.nd = ns, nd

    def mu(self, offset):
        return self.rg.h ** 2 * self.pals.absorption(desk_params(offset), self.nodes)

    def op(self, mu):
        return orc.Operator.grid(self.g, P.constant_fields(self.g, mu))


def log_array(rows):
    return np.array([[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in rows])


def test_reference_reproduces_the_committed_fixture():
    z = np.load(os.path.join(HERE, "ref_desk.npz"))
    d = Desk(int(z["n"]), int(z["n_src"]), int(z["n_det"]))
    rb = ref.Basis.init(d.rg, d.mu(0.0), d.B, int(z["k"]), float(z["tol"]))
    assert np.array_equal(rb.eigenvalues, z["eigenvalues"])
    logs = [log_array(rb.process_system(d.mu(off), d.B, float(z["tol"]), s).log)
            for s, off in enumerate(z["offsets"], start=1)]
    assert np.array_equal(np.concatenate(logs), z["log"])


@pytest.mark.parametrize("n", [9, 15, 24])
def test_operator_layout_and_blocks(n):  # grid.cpp:38-160
    d = Desk(n, 3, 2)
    assert np.array_equal(d.lay.dense(d.g.n), d.B)
    mu = d.mu(0.1)
    A_ref = d.rg.matrix(mu)
    A = d.op(mu).matrix()
    assert np.abs(A - A_ref).max() <= 2e-16 * np.abs(A_ref).max()
    assert np.array_equal(A_ref, A_ref.T)
    # full block system (grid.cpp:162-173): eliminating the boundary block gives the Schur operator
    F = d.rg.full_block_matrix(mu)
    nb = 2 * n
    S = F[nb:, nb:] - F[nb:, :nb] @ np.linalg.solve(F[:nb, :nb], F[:nb, nb:])
    assert np.abs(S - A).max() <= 1e-14 * np.abs(A).max()


def test_evenly_spaced_positions_and_errors():  # grid.cpp:107-121
    for nx, c in [(5, 1), (5, 3), (41, 8), (121, 32), (200, 198)]:
        assert ref.evenly_spaced_positions(nx, c) == P.evenly_spaced_positions(nx, c)
    for nx, c in [(5, 0), (5, 4)]:
        with pytest.raises(ref.ConfigError):
            ref.evenly_spaced_positions(nx, c)
        with pytest.raises(ValueError):
            P.evenly_spaced_positions(nx, c)
    with pytest.raises(ref.RefError):
        ref.Grid(4, 9)  # grid: nx and ny must both be at least 5
    with pytest.raises(ValueError):
        P.GridSpec.reference_2d(4, 9)


def test_normal_stream_bit_exact():  # config.cpp:249-271
    for seed in (0, 1, 1234, 20160200, 2 ** 63 + 5):
        a = ref.normal_stream(seed, 257)
        s = P.NormalStream(seed)
        b = np.array([s.next() for _ in range(257)])
        assert np.array_equal(a, b)
        assert np.array_equal(a, orc.normal_stream(seed, 257))


def test_minres_spd_and_indefinite():  # krylov.cpp:17-104, test_krylov.cpp:42-110
    rng = np.random.default_rng(5)
    n = 60
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    for eig in (np.linspace(0.5, 40, n), np.concatenate([-np.linspace(1, 5, 7), np.linspace(0.3, 30, n - 7)])):
        A = (Q * eig) @ Q.T
        A = 0.5 * (A + A.T)
        b = rng.standard_normal(n)
        xr, rr = ref.minres_dense(A, b, 1e-10, 400)
        xo, ro = orc.minres(orc.Operator.dense(A), b, 1e-10, 400)
        assert rr.converged and ro.converged
        assert rr.iterations == ro.iterations
        assert np.allclose(rr.history, ro.history, rtol=1e-6, atol=1e-16)
        assert rel(xo, xr) <= 1e-10
    # zero right-hand side: converged at once, zero solution (krylov.cpp:26-30)
    xr, rr = ref.minres_dense(A, np.zeros(n), 1e-10, 10)
    xo, ro = orc.minres(orc.Operator.dense(A), np.zeros(n), 1e-10, 10)
    assert rr.iterations == ro.iterations == 0 and rr.converged and ro.converged
    assert not xr.any() and not xo.any()


def test_from_raw_append_initial_guess():  # krylov.cpp:106-145
    d = Desk(17, 3, 3)
    mu = d.mu(0.2)
    rng = np.random.default_rng(11)
    W = rng.standard_normal((d.g.n, 7))
    AW = np.stack([d.rg.apply(mu, W[:, j]) for j in range(7)], axis=1)
    Ur, Kr = ref.from_raw(W, AW)
    rs = orc.RecycleSpace(W, AW)
    Uo, Ko = rs.UK()
    # same spaces and the same pairing A U = K, K^T K = I (column signs are the QR's)
    assert np.abs(Kr.T @ Kr - np.eye(7)).max() <= 1e-13
    assert rel(Ko @ Ko.T, Kr @ Kr.T) <= 1e-12
    assert rel(Uo @ Ko.T, Ur @ Kr.T) <= 1e-11
    b = rng.standard_normal(d.g.n)
    zr, rr = ref.initial_guess(W, AW, b)
    zo, ro = rs.initial_guess(b)
    assert rel(zo, zr) <= 1e-11 and rel(ro, rr) <= 1e-12
    # append: an independent direction is taken, a dependent one refused (krylov.cpp:117-139)
    u = rng.standard_normal(d.g.n)
    ok_r, U2, K2 = ref.from_raw_append(W, AW, u, d.rg.apply(mu, u))
    ok_o = rs.append(u, d.op(mu).apply(u))
    assert ok_r and ok_o
    Uo2, Ko2 = rs.UK()
    assert rel(Ko2 @ Ko2.T, K2 @ K2.T) <= 1e-12
    udep = W @ rng.standard_normal(7)
    ok_r, _, _ = ref.from_raw_append(W, AW, udep, AW @ np.linalg.lstsq(W, udep, rcond=None)[0])
    rs2 = orc.RecycleSpace(W, AW)
    ok_o = rs2.append(udep, AW @ np.linalg.lstsq(W, udep, rcond=None)[0])
    assert not ok_r and not ok_o


@pytest.mark.parametrize("n,k", [(11, 3), (20, 8), (31, 12)])
def test_smallest_eigenpairs(n, k):  # krylov.cpp:181-280
    d = Desk(n, 2, 2)
    mu = d.mu(0.0)
    lr, Ur = d.rg.smallest_eigenpairs(mu, k, 1e-9)
    lo, Uo = orc.smallest_eigenpairs(d.op(mu), k, 1e-9)
    assert np.allclose(lo, lr, rtol=1e-9)
    w = np.linalg.eigvalsh(d.rg.matrix(mu))[:k]
    assert np.allclose(lr, w, rtol=1e-7)
    gap = (w[-1] - w[0]) / max(1e-300, np.linalg.eigvalsh(d.rg.matrix(mu))[k] - w[-1])
    if gap < 1e3:
        assert np.linalg.svd(Uo.T @ Ur, compute_uv=False).min() >= 1 - 1e-6
    with pytest.raises(ref.ConfigError):
        d.rg.smallest_eigenpairs(mu, 0)
    with pytest.raises(orc.ConfigError):
        orc.smallest_eigenpairs(d.op(mu), 0)


def test_global_basis_refresh_append_projected():  # basis.cpp:37-112
    d = Desk(15, 3, 3)
    mu0, mu1 = d.mu(0.0), d.mu(0.25)
    rb = ref.Basis.init(d.rg, mu0, d.B, 4, 1e-8)
    V0 = rb.V
    gb = orc.GlobalBasis(V0[:, :4], V0[:, 4:])
    rb.refresh(mu1)
    gb.refresh(d.op(mu1))
    assert rel(np.abs(np.diag(gb.R)), np.abs(np.diag(rb.R))) <= 1e-10
    assert rel(gb.K_img @ gb.K_img.T, rb.K_img @ rb.K_img.T) <= 1e-11
    rng = np.random.default_rng(2)
    for t in range(4):
        y = rng.standard_normal(d.g.n)
        Ay0 = d.rg.apply(np.zeros(d.g.n), y)  # A~_* y
        assert rb.append(y, Ay0, mu1)
        assert gb.append(y, d.op(mu1).apply(y))
    b = rng.standard_normal(d.g.n)
    assert rel(gb.solve_projected(b), rb.solve_projected(b)) <= 1e-9
    assert rel(gb.projected_coordinates(b), rb.projected_coordinates(b)) <= 1e-7
    ydep = rb.V @ np.full(rb.cols, 0.3)  # test_basis.cpp:110-121
    assert not rb.append(ydep, d.rg.apply(np.zeros(d.g.n), ydep), mu1)
    assert not gb.append(ydep, d.op(mu1).apply(ydep))
    assert rb.cols == gb.cols


def test_refresh_drops_dependent_column():  # basis.cpp:56-75
    d = Desk(15, 3, 3)
    mu0 = d.mu(0.0)
    rb0 = ref.Basis.init(d.rg, mu0, d.B, 4, 1e-8)
    V = rb0.V
    X0 = V[:, 4:].copy()
    X0[:, 3] = X0[:, 1] * 2.0 - X0[:, 0]  # a dependent initial-solution column
    rb = ref.Basis.init_from(d.rg, V[:, :4], X0)
    gb = orc.GlobalBasis(V[:, :4], X0)
    rb.refresh(mu0)
    gb.refresh(d.op(mu0))
    assert rb.cols == gb.cols == V.shape[1] - 1
    assert np.array_equal(rb.markers, gb.markers)
    assert rel(gb.V, rb.V) <= 1e-15


def test_process_system_error_behaviour():  # basis.cpp:186-188
    d = Desk(15, 3, 3)
    rb = ref.Basis.init(d.rg, d.mu(0.0), d.B, 4, 1e-8)
    V = rb.V
    gb = orc.GlobalBasis(V[:, :4], V[:, 4:])
    mu = d.mu(0.4)
    with pytest.raises(ref.SolverError) as er:
        rb.process_system(mu, d.B, 1e-8, 1, maxit=3)
    with pytest.raises(orc.SolverError) as eo:
        orc.process_system(gb, d.op(mu), d.lay, 1e-8, 1, 3, orc.MINRES)
    assert "correction solve failed at system 1, rhs 0" in str(er.value)
    assert "correction solve failed at system 1, rhs 0" in str(eo.value)


@pytest.mark.parametrize("n,ns,nd,k,tol", [(17, 3, 3, 5, 1e-8), (25, 5, 4, 8, 1e-7)])
def test_build_sequence_lockstep(n, ns, nd, k, tol):  # basis.cpp:136-266
    """init_basis + six systems on both sides, each from its own seed, plus
    the per-RHS-only comparator: identical BuildLogs."""
    d = Desk(n, ns, nd)
    mu0 = d.mu(0.0)
    rb = ref.Basis.init(d.rg, mu0, d.B, k, tol)
    gb, X0, lam, U0 = orc.init_basis(d.op(mu0), d.op(mu0), d.lay, k, tol, orc.MINRES)
    assert np.allclose(lam, rb.eigenvalues, rtol=1e-9)
    Vr = rb.V
    rrec = ref.PerRhsRecycler(d.rg, Vr[:, :k], Vr[:, k:])
    orec = orc.PerRhsRecycler(U0, X0)
    for s, off in enumerate([0.02, 0.05, 0.02, 0.11, 0.4, 0.0], start=1):
        mu = d.mu(off)
        a, b = rb.process_system(mu, d.B, tol, s), orc.process_system(gb, d.op(mu), d.lay, tol, s, 0, orc.MINRES)
        la, lb = log_array(a.log), log_array(b.log)
        assert np.array_equal(la[:, [0, 1, 3, 4]], lb[:, [0, 1, 3, 4]]), (s, la[:, 3], lb[:, 3])
        assert np.allclose(la[:, 2], lb[:, 2], rtol=1e-5)
        assert rel(b.X, a.X) <= 1e-9
        assert rb.cols == gb.cols
        a, b = rrec.solve_system(mu, d.B, tol, s), orec.solve_system(d.op(mu), d.lay, tol, s, 0, orc.MINRES)
        la, lb = log_array(a.log), log_array(b.log)
        assert np.array_equal(la[:, [0, 1, 3, 4]], lb[:, [0, 1, 3, 4]])
        assert rel(b.X, a.X) <= 1e-9
    assert [rb.space(j) for j in range(ns + nd)] == [gb.space(j) for j in range(ns + nd)]
    assert np.array_equal(rb.markers, gb.markers)


def test_romb_files_interchange(tmp_path):  # io.cpp:77-131
    """A basis written by the reference reads back bit for bit through the
    product's reader, and the other way round (host code: no GPU needed)."""
    from paper_1602_00138_b200 import romdot as R
    rng = np.random.default_rng(8)
    V = np.asfortranarray(rng.standard_normal((37, 5)))
    mk = np.array([0, 0, 1, 1, 2], dtype=np.uint8)
    p1, p2 = str(tmp_path / "ref.romb"), str(tmp_path / "ours.romb")
    ref.write_basis(p1, V, mk)
    R.romb_write(p2, V, mk)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    V1, m1 = R.romb_read(p1)
    V2, m2 = ref.read_basis(p2)
    assert V1.tobytes(order="F") == V.tobytes(order="F") == V2.tobytes(order="F")
    assert list(m1) == list(m2) == list(mk)
    open(p1, "wb").write(open(p1, "rb").read()[:-3])  # truncated file: IoError on both sides
    with pytest.raises(ref.IoError):
        ref.read_basis(p1)
    with pytest.raises(R.IoError):
        R.romb_read(p1)


def test_format_sci():  # io.cpp:11-15
    from paper_1602_00138_b200 import offline as O
    for v in (0.0, 1e-7, 1.23456789e-3, -4.5e10, 1.0):
        assert ref.format_sci(v) == O.format_sci(v)


def test_criterion5_reference_passes_its_own_bar(tmp_path):  # acceptance.cpp:314-334 (smaller grid: seconds)
    cfg = ref.exp_config(nx=61, ny=61, n_src=16, n_det=16, m_bumps=9, seed=1234)
    ours, base = ref.compare_recycling(cfg, str(tmp_path))
    n, nrhs, _ = ref.exp_dims(cfg)
    g = P.GridSpec.reference_2d(61, 61)
    lay = P.make_layout(g, (16,), (16,), src_high=True)
    mus = [ref.exp_mu(cfg, i)[0] for i in range(3)]
    op = lambda mu: orc.Operator.grid(g, P.constant_fields(g, mu))  # noqa: E731
    gb, X0, lam, U0 = orc.init_basis(op(mus[0]), op(mus[0]), lay, 10, 1e-7, orc.MINRES)
    rec = orc.PerRhsRecycler(U0, X0)
    o = b = 0
    for s in (1, 2):
        o += orc.process_system(gb, op(mus[s]), lay, 1e-7, s, 0, orc.MINRES).inner_iterations
        b += rec.solve_system(op(mus[s]), lay, 1e-7, s, 0, orc.MINRES).inner_iterations
    assert abs(o - ours) <= 2 and abs(b - base) <= 2, (o, ours, b, base)
    assert (ours * 2 <= base) == (o * 2 <= b)
