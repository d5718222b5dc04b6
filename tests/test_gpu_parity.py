"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (SURVEY.md App. C protocol).

Tolerances (fp64):
  * stencil apply            <= 1e-14 relative (entrywise vs max |y|)
  * projections / QR          <= 1e-12 relative
  * solves                    iterations within +-2 of the oracle per solve,
                              explicit residual <= tol for every solution
  * basis observables         reduced transfer within 1e-8 relative
"""
import numpy as np
import pytest

import oracle as orc
from helpers import Desk, rom_transfer
from paper_1602_00138_b200 import problem as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_1602_00138_b200 import build, romdot
    build.build()
    return romdot


def random_fields(grid, seed):
    rng = np.random.default_rng(seed)
    return P.Fields(D=rng.uniform(0.3, 0.4, grid.n), mu=grid.h ** 2 * rng.uniform(0.005, 0.05, grid.n), shift=0.0)


@pytest.mark.parametrize("d,N", [(2, (37, 29)), (3, (11, 9, 13)), (2, (317, 317)), (3, (47, 47, 47)),
                                 (2, (64, 30)), (3, (48, 40, 44)), (3, (34, 17, 70))])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("ncols", [1, 3, 9])
def test_stencil_matches_oracle(rd, d, N, cplx, ncols):
    """ncols = 1: the z-marching one-column kernel; ncols >= 2: the TMA-staged
    multi-column kernel (stencil_tma.cuh; NC = 4 complex / 8 real columns per
    block with a ragged last group), except float64 with odd N0 (row pitch not
    16-byte aligned), which keeps the one-column kernel. Odd N0 complex uses
    the row-padded coefficient copy."""
    g = P.GridSpec(d=d, N=N, h=1.0 / (N[0] - 1), D_bg=0.33)
    f = random_fields(g, 5)
    if cplx:
        f = P.Fields(f.D, f.mu, shift=g.h ** 2 * 0.1)
    dt = np.complex128 if cplx else np.float64
    rng = np.random.default_rng(6)
    x = rng.standard_normal((g.n, ncols))
    if cplx:
        x = x + 1j * rng.standard_normal((g.n, ncols))
    y_ref = orc.Operator.grid(g, f, dt).apply(x)
    y = rd.SchurOperator(g, f, dt).apply(x)
    assert np.abs(y - y_ref).max() <= 1e-14 * np.abs(y_ref).max()


@pytest.mark.parametrize("d,N", [(3, (48, 40, 44)), (2, (317, 317)), (3, (47, 47, 47))])
@pytest.mark.parametrize("cplx", [False, True])
def test_multicolumn_stencil_bitwise_equals_one_column(rd, d, N, cplx):
    """The multi-column kernels keep zmarch's loads, products and summation
    order per column, so a 13-column apply equals 13 one-column applies bit
    for bit (same for the opt-in four-column kernel, ROMDOT_STENCIL_MC=1, run
    in a subprocess because the switch is read once per process)."""
    g = P.GridSpec(d=d, N=N, h=1.0 / (N[0] - 1), D_bg=0.33)
    f = random_fields(g, 5)
    if cplx:
        f = P.Fields(f.D, f.mu, shift=g.h ** 2 * 0.1)
    dt = np.complex128 if cplx else np.float64
    rng = np.random.default_rng(9)
    x = rng.standard_normal((g.n, 13))
    if cplx:
        x = x + 1j * rng.standard_normal((g.n, 13))
    op = rd.SchurOperator(g, f, dt)
    ym = op.apply(x)
    y1 = np.stack([op.apply(np.ascontiguousarray(x[:, j])) for j in range(13)], axis=1)
    assert np.array_equal(ym, y1)


def test_four_column_stencil_opt_in(rd, tmp_path):
    """ROMDOT_STENCIL_MC=1 (with the TMA kernel off) runs stencil_kernel_mc:
    3 / 9 columns (ragged last group of 4), 2D and 3D, and 50 groups on a
    long z axis. (Its grid-chunking branch needs > 65535 blocks in z, which
    stencil_kz's sizing only reaches at ~2.6e5 columns: not exercised.)"""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "ROOT"); sys.path.insert(0, "ROOT/oracle")
import oracle as orc
from paper_1602_00138_b200 import problem as P, romdot as R
for d, N, nc in [(3, (11, 9, 13), 3), (3, (11, 9, 13), 9), (2, (37, 29), 9), (3, (8, 8, 2000), 200)]:
    g = P.GridSpec(d=d, N=N, h=1.0 / (N[0] - 1), D_bg=0.33)
    rng = np.random.default_rng(5)
    f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=g.h ** 2 * rng.uniform(0.005, 0.05, g.n), shift=g.h ** 2 * 0.1)
    x = rng.standard_normal((g.n, nc)) + 1j * rng.standard_normal((g.n, nc))
    y = R.SchurOperator(g, f, np.complex128).apply(x)
    yr = orc.Operator.grid(g, f, np.complex128).apply(x)
    assert np.abs(y - yr).max() <= 1e-14 * np.abs(yr).max(), (d, N, nc)
print("ok")
'''.replace("ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    env = dict(os.environ, ROMDOT_STENCIL_MC="1", ROMDOT_STENCIL_TMA="0")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def _problem(cfg_name, point=1, omega=0.0):
    c = P.CONFIGS[cfg_name]
    return c, c.grid, c.layout(), c.fields(point, omega)


@pytest.mark.parametrize("cfg,omega", [("T2", 0.0), ("T3", 0.0), ("T2c", 0.2)])
def test_plain_cg_matches_oracle(rd, cfg, omega):
    c, g, lay, f = _problem(cfg, 1, omega)
    dt = c.dtype
    B = lay.dense(g.n, dt)
    op_o = orc.Operator.grid(g, f, dt)
    op_g = rd.SchurOperator(g, f, dt)
    A = op_o.matrix() if g.n <= 2000 else None
    for j in range(lay.n_rhs):
        b = B[:, j]
        ro = orc.recycled_cg(op_o, None, b, 0.25e-8, 2 * g.n)
        rg = rd.recycled_cg(op_g, None, None, b, 0.25e-8, 2 * g.n)
        assert rg.report.converged
        assert abs(rg.report.iterations - ro.report.iterations) <= 2
        x = rg.correction
        res = op_o.apply(x)
        assert np.linalg.norm(b - res) <= 0.25e-8 * np.linalg.norm(b) * 1.01
        assert np.linalg.norm(x - ro.correction) <= 1e-6 * np.linalg.norm(ro.correction)


@pytest.mark.parametrize("cfg,omega", [("T2", 0.0), ("T2c", 0.2), ("T3", 0.0)])
def test_recycled_cg_matches_oracle(rd, cfg, omega):
    c, g, lay, f = _problem(cfg, 1, omega)
    dt = c.dtype
    rng = np.random.default_rng(11)
    op_o = orc.Operator.grid(g, f, dt)
    W = rng.standard_normal((g.n, 9)).astype(dt)
    AW = op_o.apply(W)
    rs = orc.RecycleSpace(W, AW)
    U, K = rs.UK()
    # device from_raw reproduces the oracle's space (projector and A U = K)
    Ug, Kg = rd.recycle_space_from_raw(W, AW)
    Pg = Kg @ Kg.T
    Po = K @ K.T
    assert np.abs(Pg - Po).max() <= 1e-12
    assert np.linalg.norm(op_o.apply(Ug) - Kg) <= 1e-10 * np.linalg.norm(Kg)
    assert np.linalg.norm(Kg.T @ Kg - np.eye(9)) <= 1e-12
    b = lay.dense(g.n, dt)[:, 0]
    _, r0 = rs.initial_guess(b)
    ro = orc.recycled_cg(op_o, rs, r0, 1e-9, 2 * g.n, np.linalg.norm(b))
    rg = rd.recycled_cg(rd.SchurOperator(g, f, dt), U, K, r0, 1e-9, 2 * g.n, np.linalg.norm(b))
    assert rg.report.converged
    assert abs(rg.report.iterations - ro.report.iterations) <= 2
    assert np.linalg.norm(r0 - op_o.apply(rg.correction)) <= 1.01e-9 * np.linalg.norm(b)
    assert np.linalg.norm(rg.image - op_o.apply(rg.new_direction)) <= 1e-12 * np.linalg.norm(rg.image)


def _shared_seed(c, g, lay):
    """U0, X0 from the oracle so both builds start from identical bytes."""
    f0 = c.fields(0)
    op0r = orc.Operator.grid(g, f0)
    op0 = orc.Operator.grid(g, f0, c.dtype)
    lam, U0 = orc.smallest_eigenpairs(op0r, c.k, min(c.tol, 1e-8))
    X0, _ = orc.initial_solutions(op0, lay, c.tol)
    return U0.astype(c.dtype), X0


@pytest.mark.parametrize("cfg", ["T2", "T2c", "T3", "T3c"])
def test_process_system_lockstep_parity(rd, cfg):
    c = P.CONFIGS[cfg]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    gb_o = orc.GlobalBasis(U0, X0, c.cap)
    gb_g = rd.GlobalBasis(U0, X0, c.cap)
    B = lay.dense(g.n, c.dtype)
    flips = 0
    total = 0
    for s, (pt, w) in enumerate(c.systems(), start=1):
        f = c.fields(pt, w)
        op_o = orc.Operator.grid(g, f, c.dtype)
        op_g = rd.SchurOperator(g, f, c.dtype)
        po = orc.process_system(gb_o, op_o, lay, c.tol, s)
        pg = rd.process_system(gb_g, op_g, lay, c.tol, s)
        # explicit residual for every GPU solution (test_basis.cpp:180-193)
        R = op_o.apply(pg.X) - B
        for j in range(lay.n_rhs):
            assert np.linalg.norm(R[:, j]) <= c.tol * np.linalg.norm(B[:, j])
        for ro, rg in zip(po.log, pg.log):
            total += 1
            if ro.appended != rg.appended or (ro.iterations == 0) != (rg.iterations == 0):
                flips += 1
                continue
            assert abs(ro.iterations - rg.iterations) <= 2, (s, ro, rg)
            assert ro.init_relres == pytest.approx(rg.init_relres, rel=1e-6, abs=1e-13)
        assert gb_g.cols == gb_o.cols or flips
        if flips:
            break  # free-running builds diverge after a decision flip (App. C.2)
    assert flips <= max(1, total // 20)
    # basis-invariant observable: reduced transfer at the last system
    A = op_o.matrix() if g.n <= 2500 else None
    if A is not None and not flips:
        Bt, Ct = B[:, : lay.n_src], B[:, lay.n_src:]
        to = rom_transfer(gb_o.V, A, Bt, Ct)
        tg = rom_transfer(gb_g.V, A, Bt, Ct)
        assert np.linalg.norm(to - tg) <= 1e-8 * np.linalg.norm(to)


def test_refresh_factorisation_properties(rd):
    d = Desk(15, 3, 3)
    op_o = d.op(0.0)
    U0 = np.linalg.qr(np.random.default_rng(1).standard_normal((d.grid.n, 4)))[0]
    X0, _ = orc.initial_solutions(op_o, d.layout, 1e-8)
    gb = rd.GlobalBasis(U0, X0)
    # before the first refresh the image factor is empty, as the reference's
    # default-constructed Kimg_ / R_ (include/romdot/basis.hpp:63)
    assert not gb.factored
    assert gb.K_img.shape == (d.grid.n, 0) and gb.R.shape == (0, 0) and gb.W.shape == (d.grid.n, 0)
    op = rd.SchurOperator(d.grid, P.constant_fields(d.grid, d.mu_of(0.0)))
    gb.refresh(op)
    assert gb.factored
    A = op_o.matrix()
    Kf = A @ gb.V
    K, R = gb.K_img, gb.R
    r = gb.cols
    assert np.linalg.norm(K @ R - Kf) <= 1e-12 * np.linalg.norm(Kf)
    assert np.linalg.norm(K.T @ K - np.eye(r)) <= 1e-12
    assert np.all(np.tril(R, -1) == 0)
    assert np.linalg.norm(A @ gb.W - K) <= 1e-10 * np.linalg.norm(K)
    rng = np.random.default_rng(4)
    for t in range(5):
        y = rng.standard_normal(d.grid.n)
        assert gb.append(y, A @ y)
    y = gb.V @ np.full(gb.cols, 0.3)
    assert not gb.append(y, A @ y)
    b = rng.standard_normal(d.grid.n)
    x = gb.solve_projected(b)
    c, *_ = np.linalg.lstsq(A @ gb.V, b, rcond=None)
    assert np.linalg.norm(x - gb.V @ c) <= 1e-8 * np.linalg.norm(x)
    assert np.allclose(gb.projected_coordinates(b), c, rtol=1e-6, atol=1e-10 * np.abs(c).max())


def test_build_is_bitwise_deterministic(rd):
    c = P.CONFIGS["T2"]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)

    def build():
        gb = rd.GlobalBasis(U0, X0)
        f = c.fields(1)
        rd.process_system(gb, rd.SchurOperator(g, f), lay, c.tol, 1)
        return gb.V

    assert build().tobytes() == build().tobytes()


@pytest.mark.parametrize("cfg", ["T2", "T3"])
def test_device_eigen_seed_matches_oracle(rd, cfg):
    """smallest_eigenpairs (krylov.cpp:181-280): eigenvalues vs the oracle
    (exact shift-invert) to 1e-8 relative; residuals <= tol * lambda_max."""
    c = P.CONFIGS[cfg]
    g = c.grid
    f0 = c.fields(0)
    lam_o, U_o = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, 1e-8)
    op = rd.SchurOperator(g, f0)
    lam, U = rd.smallest_eigenpairs(op, c.k, 1e-8)
    assert np.allclose(lam, lam_o, rtol=1e-8)
    A = orc.Operator.grid(g, f0)
    lm = A.lam_max
    for i in range(c.k):
        r = A.apply(U[:, i]) - lam[i] * U[:, i]
        assert np.linalg.norm(r) <= 1e-8 * lm
    assert np.linalg.norm(U.T @ U - np.eye(c.k)) <= 1e-7


@pytest.mark.parametrize("m,want,n", [(64, 64, 4000), (256, 219, 4000), (1024, 219, 16384)])
def test_rrqr_known_rank_decay_09(rd, m, want, n):
    """C5 RRQR shapes at small n: A = Q diag(0.9^j) P (seeded permutation),
    rank at 1e-10 is 64 / 219 / 219; same rank, R diagonal and
    retained span (principal angles) as the oracle's Householder QRCP -- the
    m = 1024 case runs the multi-level path (805 columns dropped below tol)."""
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((n, m)))
    A = (Q * (0.9 ** np.arange(m)))[:, rng.permutation(m)]
    rk, perm, rdiag, Qg = rd.rrqr(A, 1e-10, normalize=False)
    ro, permo, rdo, Qo = orc.qrcp(A, 1e-10, normalize=False)
    assert rk == want == ro
    assert np.allclose(rdiag[:rk], rdo[:rk], rtol=1e-6)
    assert np.linalg.norm(Qg.T @ Qg - np.eye(rk)) <= 1e-12
    # principal angles between retained spaces
    s = np.linalg.svd(Qo.T @ Qg, compute_uv=False)
    assert np.sqrt(max(0.0, 1.0 - s.min() ** 2)) <= 1e-6


@pytest.mark.parametrize("cplx", [False, True])
def test_rrqr_candidate_basis_matches_oracle(rd, cplx):
    """Compression of a real build's candidate basis (column-normalised, App. A9):
    identical rank to the oracle QRCP and the same retained span on sigma >= 1e-6."""
    c = P.CONFIGS["T2c" if cplx else "T2"]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    gb = orc.GlobalBasis(U0, X0, c.cap)
    for s, (pt, w) in enumerate(c.systems(), start=1):
        orc.process_system(gb, orc.Operator.grid(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
    V = gb.V
    rk, perm, rdiag, Qg = rd.rrqr(V, 1e-10, normalize=True)
    ro, permo, rdo, Qo = orc.qrcp(V, 1e-10, normalize=True)
    assert rk == ro
    # pivot order is not unique here (every normalised column starts tied at norm 1),
    # so R diagonals differ between valid QRCP runs; rank and span are the invariants
    assert rdiag[0] == pytest.approx(1.0) and np.all(rdiag[:rk] > 1e-10)
    assert np.linalg.norm(Qg.conj().T @ Qg - np.eye(rk)) <= 1e-10
    # angles restricted to the well-determined part of the spectrum (App. C.1)
    Un, sn, _ = np.linalg.svd(V / np.linalg.norm(V, axis=0), full_matrices=False)
    keep = sn >= 1e-6 * sn[0]
    Ut = Un[:, keep]
    for Qx in (Qg, Qo):
        s = np.linalg.svd(Qx.conj().T @ Ut, compute_uv=False)
        assert np.sqrt(max(0.0, 1.0 - s.min() ** 2)) <= 1e-6


def test_build_deterministic_across_interleaved_builds(rd):
    """Bitwise reproducibility (test_basis.cpp:210-223) must survive other builds
    running in between (allocation reuse, cache state): T2c built 4 times with T3c
    builds interleaved gives identical BuildLogs and V."""
    c = P.CONFIGS["T2c"]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    c3 = P.CONFIGS["T3c"]
    z3 = _shared_seed(c3, c3.grid, c3.layout())

    def build(cfg, U, X):
        gb = rd.GlobalBasis(U, X, cfg.cap)
        rows = []
        for s, (pt, w) in enumerate(cfg.systems(), start=1):
            pr = rd.process_system(gb, rd.SchurOperator(cfg.grid, cfg.fields(pt, w), cfg.dtype), cfg.layout(),
                                   cfg.tol, s)
            rows += [(r.init_relres, r.iterations, r.appended) for r in pr.log]
        return rows, gb.V

    ref_rows, ref_V = build(c, U0, X0)
    for rep in range(3):
        build(c3, *z3)
        rows, V = build(c, U0, X0)
        assert rows == ref_rows
        assert V.tobytes() == ref_V.tobytes()


def test_device_residual_norms_match_numpy(rd):
    c = P.CONFIGS["T3c"]
    g, lay = c.grid, c.layout()
    f = c.fields(1, 0.1)
    op_o = orc.Operator.grid(g, f, c.dtype)
    rng = np.random.default_rng(3)
    X = (rng.standard_normal((g.n, lay.n_rhs)) + 1j * rng.standard_normal((g.n, lay.n_rhs))).astype(c.dtype)
    B = lay.dense(g.n, c.dtype)
    want = np.linalg.norm(op_o.apply(X) - B, axis=0) / np.linalg.norm(B, axis=0)
    got = rd.residual_norms(rd.SchurOperator(g, f, c.dtype), lay, X)
    assert np.allclose(got, want, rtol=1e-12)


def test_basis_compress_in_place(rd):
    c = P.CONFIGS["T2"]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    gb = rd.GlobalBasis(U0, X0)
    for s, (pt, w) in enumerate(c.systems(), start=1):
        rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w)), lay, c.tol, s)
    V = gb.V
    ro, *_ = orc.qrcp(V, 1e-10, normalize=True)
    rank, perm, rdiag = gb.compress(1e-10)
    assert rank == ro == gb.cols
    Q = gb.V
    assert np.linalg.norm(Q.T @ Q - np.eye(rank)) <= 1e-10
    Vn = V / np.linalg.norm(V, axis=0)
    Un, sn, _ = np.linalg.svd(Vn, full_matrices=False)
    Ut = Un[:, sn >= 1e-6 * sn[0]]
    s = np.linalg.svd(Q.T @ Ut, compute_uv=False)
    assert np.sqrt(max(0.0, 1 - s.min() ** 2)) <= 1e-6


@pytest.mark.parametrize("cfg", ["T2", "T3c"])
def test_per_rhs_recycler_lockstep_parity(rd, cfg):
    """BaselinePerRhsRecycler (basis.cpp:209-266) on the device vs the CPU
    checker from identical U0/X0: every log row (±2 iterations, same append
    decisions, init_relres), explicit residual <= tol (test_basis.cpp:225-240)."""
    c = P.CONFIGS[cfg]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    po_ = orc.PerRhsRecycler(U0, X0)
    pg_ = rd.PerRhsRecycler(U0, X0)
    B = lay.dense(g.n, c.dtype)
    appends = 0
    for s, (pt, w) in enumerate(c.systems(), start=1):
        f = c.fields(pt, w)
        op_o = orc.Operator.grid(g, f, c.dtype)
        po = po_.solve_system(op_o, lay, c.tol, s)
        pg = pg_.solve_system(rd.SchurOperator(g, f, c.dtype), lay, c.tol, s)
        R = op_o.apply(pg.X) - B
        assert (np.linalg.norm(R, axis=0) <= c.tol * np.linalg.norm(B, axis=0)).all()
        for ro, rg in zip(po.log, pg.log):
            assert ro.appended == rg.appended, (s, ro, rg)
            assert abs(ro.iterations - rg.iterations) <= 2, (s, ro, rg)
            assert ro.init_relres == pytest.approx(rg.init_relres, rel=1e-6, abs=1e-13)
        appends += pg.appends
    # V = [U0, X0, every RHS's own directions]; U_j = [U0, X0_j, own directions]
    assert pg_.cols == c.k + lay.n_rhs + appends
    assert sum(len(pg_.space(j)) for j in range(lay.n_rhs)) == lay.n_rhs * (c.k + 1) + appends


@pytest.mark.parametrize("cfg,ours_ref,base_ref,bar", [("R5", 4941, 9634, 0.6), ("R5b", 4098, 9887, 0.5)])
def test_global_basis_beats_per_rhs_recycling(rd, cfg, ours_ref, base_ref, bar):
    """Acceptance criterion 5 (acceptance.cpp:314-334, cmd_compare_recycling
    harness.cpp:209-252) on R5, its 121^2 / 32+32 / k_eig 10 / tol 1e-7 mirror
    with the reference's parameter sequence: the shared-basis build needs
    about half the inner iterations of per-RHS-only recycling. The reference
    asserts ours * 2 <= baseline (<= 0.5) on its PaLS desk phantom, which is
    not in the repository. The ratio depends on the phantom: over
    12 seeds of this generator the CPU checker gives 0.32 .. 0.69 (median
    0.59). So the test pins the device to the checker's own counts (+-2 per
    row) and applies the reference's <= 0.5 bar where the checker meets it
    (R5b, seed 20160209: 0.414); on the default seed (R5: 0.513 on the
    checker, MINRES 0.53) the bar is 0.6."""
    c = P.CONFIGS[cfg]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    gb = rd.GlobalBasis(U0, X0, c.cap)
    pr = rd.PerRhsRecycler(U0, X0)
    ours = base = 0
    for s, (pt, w) in enumerate(c.systems()[:2], start=1):
        f = c.fields(pt, w)
        ours += rd.process_system(gb, rd.SchurOperator(g, f, c.dtype), lay, c.tol, s, want_X=False).inner_iterations
        base += pr.solve_system(rd.SchurOperator(g, f, c.dtype), lay, c.tol, s, want_X=False).inner_iterations
    assert ours / base <= bar, (ours, base)
    assert abs(ours - ours_ref) <= 2 * 128 and abs(base - base_ref) <= 2 * 128, (ours, base)


def test_full_config_parity_C1(rd):
    """BASELINE configs[0] (C1, 2D 129^2, 32 RHS, 4 systems) at full size
    against the CPU checker with north_star's tolerances: lockstep BuildLog
    (+/-2 iterations, same append decisions), residual <= tol per solve, same
    RRQR rank, principal-angle sine <= 1e-6, ROM transfer / Jacobian <= 1e-8."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "parity_full", os.path.join(os.path.dirname(__file__), "..", "scripts", "parity_full.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    out = mod.run("C1")
    assert out["pass"], out


def test_partial_lockstep_device_seed_C2(rd):
    """The target-config recipe (scripts/parity_full.py --rhs --device-seed, run
    at C4 on the box) on the complex 2D config C2: device U0 / X0 checked with
    the checker's operator, then the first 4 RHS of two systems (omega = 0 and
    0.05) in lockstep with north_star's tolerances."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "parity_full", os.path.join(os.path.dirname(__file__), "..", "scripts", "parity_full.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    out = mod.run("C2", n_systems=2, n_rhs=4, device_seed=True)
    assert out["X0_max_explicit_residual"] <= out["tol"], out
    assert out["eig_residual_over_lammax"] <= 1e-8, out
    assert out["pass"], out


@pytest.mark.parametrize("d,N,cplx,width", [
    (3, (64, 64, 64), False, 40),   # C3 grid: many steps per CTA, plane lag L > 1
    (3, (48, 40, 44), True, 20),    # non-cubic complex, ragged last step
    (2, (317, 317), True, 33),      # 2D: lag of one x-line
    (3, (12, 12, 12), True, 9),     # tiny: fewer tiles than SMs, one step
    (2, (33, 33), False, 6),
    (3, (64, 64, 64), True, 72),    # the widths C4 runs (c = 65..81): 10 columns per consumer warp
    (3, (64, 64, 64), True, 96),    # 12 columns per warp
    (3, (64, 64, 64), True, 128),   # the widest instantiation (16 per warp)
])
def test_fused_iteration_matches_unfused(rd, monkeypatch, d, N, cplx, width):
    """cg_fused (update of iteration i + stencil/dots/K^T w of i+1 in one launch,
    cg_fused.cuh) against the three-launch iteration on the same solve: both
    converge, residual histories equal to rounding over the first iterations,
    explicit residual <= tol. The random recycle spaces make these solves rough
    (residual jumps of 20x), so the two roundings drift apart later; the
    iteration counts are held to 2% + 2."""
    g = P.GridSpec(d=d, N=N, h=1.0 / (N[0] - 1), D_bg=0.33)
    f = random_fields(g, 8)
    dt = np.complex128 if cplx else np.float64
    if cplx:
        f = P.Fields(f.D, f.mu, shift=g.h ** 2 * 0.1)
    op_o = orc.Operator.grid(g, f, dt)
    rng = np.random.default_rng(21)
    # real W (also for the complex operator): a complex random W makes the
    # bilinear K^T K = I basis ill-conditioned and COCG plateaus on both paths
    W = rng.standard_normal((g.n, width)).astype(dt)
    U, K = rd.recycle_space_from_raw(W, op_o.apply(W))
    b = rng.standard_normal(g.n).astype(dt)
    r0 = b - K @ (K.T @ b)
    tol = 1e-8
    op_g = rd.SchurOperator(g, f, dt)
    out = {}
    for fused in ("0", "1"):
        monkeypatch.setenv("ROMDOT_FUSED", fused)
        out[fused] = rd.recycled_cg(op_g, U, K, r0, tol, 2 * g.n, np.linalg.norm(b))
    a, c = out["0"], out["1"]
    assert a.report.converged and c.report.converged
    assert abs(a.report.iterations - c.report.iterations) <= 2 + 0.02 * a.report.iterations
    m = min(10, len(a.report.rel_residual_history), len(c.report.rel_residual_history))
    assert np.allclose(c.report.rel_residual_history[:m], a.report.rel_residual_history[:m], rtol=1e-8, atol=0)
    for res in (a, c):
        assert np.linalg.norm(r0 - op_o.apply(res.correction)) <= 1.01 * tol * np.linalg.norm(b)
    assert np.linalg.norm(c.correction - a.correction) <= 1e-5 * np.linalg.norm(a.correction)


def test_fused_iteration_protocol_check(rd):
    """Race check of cg_fused's cross-CTA protocol (compute-sanitizer is closed
    on the GPU pool): with ROMDOT_FUSED_CHECK=1 every stencil halo read verifies
    that the tiles it reads carry the current launch's epoch, stamped by the
    owning CTA's update warp and published by the same release chain as r'.
    Runs the T3c build and a C3-grid fused solve (many steps per CTA, plane lag
    L > 1) in a subprocess; any stale read fails the solve."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "ROOT")
from paper_1602_00138_b200 import problem as P, romdot as R
ctx = R.default_context()
for name in ("T3c", "C3"):
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    f0 = c.fields(0)
    lam, U0 = R.smallest_eigenpairs(R.SchurOperator(g, f0, np.float64), c.k, 1e-8)
    X0, _ = R.initial_solutions(R.SchurOperator(g, f0, c.dtype), lay, c.tol)
    gb = R.GlobalBasis(U0.astype(c.dtype), X0, c.cap)
    for s, (pt, w) in enumerate(c.systems()[:2], start=1):
        R.process_system(gb, R.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s, want_X=False)
checked, bad = ctx.fused_check()
print("checked", checked, "violations", bad)
assert checked > 1000 and bad == 0
'''.replace("ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    env = dict(os.environ, ROMDOT_FUSED_CHECK="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-3000:])


# ---- batched correction solves after the candidate cap (bcg_defl.cuh) ----
# Once the cap stops the appends the reference's loop (basis.cpp:168-205) leaves the
# remaining right-hand sides independent; the device then runs 8 solves at a time with
# the system's eigen block streamed once for all of them. Same BuildLog as the one-solve
# path and as the CPU checker.
@pytest.mark.parametrize("d,N,k,cplx,nsd,cap_extra", [
    (3, 20, 12, True, (2, 3), 4),     # complex, eigen block 12 (2 column tiles, one ragged), 12 RHS
    (2, 48, 20, False, (9,), 6),      # real 2D, eigen block 20, 18 RHS (more than two batches)
    (3, 24, 40, True, (3, 3), 10),    # complex, eigen block 40 (DMMA steps 16 with a ragged tail), 18 RHS
    (2, 40, 6, True, (5,), 3),        # one ragged column tile
])
def test_batched_tail_matches_one_solve_path_and_oracle(rd, monkeypatch, d, N, k, cplx, nsd, cap_extra):
    nrhs = 2 * int(np.prod(nsd))
    c = P.ProblemConfig("bt", d=d, N=N, n_src=nsd, n_det=nsd, m_rbf=4, n_points=2,
                        omegas=(0.0, 0.1) if cplx else (0.0,), k=k, complex=cplx, cap=k + nrhs + cap_extra)
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    B = lay.dense(g.n, c.dtype)
    runs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("ROMDOT_BATCH", mode)
        gb = rd.GlobalBasis(U0, X0, c.cap)
        out = []
        for s, (pt, w) in enumerate(c.systems(), start=1):
            out.append(rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s))
        runs[mode] = (out, gb.batched_solves, gb.cols)
    (seq, nb0, cols0), (bat, nb1, cols1) = runs["0"], runs["1"]
    assert nb0 == 0 and nb1 >= 8, (nb0, nb1)         # the batched iteration really ran
    assert cols0 == cols1 == c.cap
    gbo = orc.GlobalBasis(U0, X0, c.cap)
    for s, (pt, w) in enumerate(c.systems(), start=1):
        a, b = seq[s - 1], bat[s - 1]
        op_o = orc.Operator.grid(g, c.fields(pt, w), c.dtype)
        po = orc.process_system(gbo, op_o, lay, c.tol, s)
        for ra, rb, ro in zip(a.log, b.log, po.log):
            assert (ra.system, ra.rhs, ra.appended) == (rb.system, rb.rhs, rb.appended) == (ro.system, ro.rhs, ro.appended)
            assert abs(ra.iterations - rb.iterations) <= 1 and abs(rb.iterations - ro.iterations) <= 2, (ra, rb, ro)
            assert rb.init_relres == pytest.approx(ra.init_relres, rel=1e-9, abs=1e-14)
            assert rb.init_relres == pytest.approx(ro.init_relres, rel=1e-6, abs=1e-13)
        assert np.linalg.norm(b.X - a.X) <= 1e-9 * np.linalg.norm(a.X)
        assert np.linalg.norm(b.X - po.X) <= 1e-6 * np.linalg.norm(po.X)
        R = op_o.apply(b.X) - B
        assert (np.linalg.norm(R, axis=0) <= c.tol * np.linalg.norm(B, axis=0)).all()


def test_batched_tail_is_bitwise_deterministic(rd):
    """Two capped builds give byte-identical solutions and BuildLogs (test_basis.cpp:210-223):
    a slot's arithmetic does not depend on what the other slots hold."""
    c = P.CONFIGS["T3c"]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    outs = []
    for _ in range(2):
        gb = rd.GlobalBasis(U0, X0, c.cap)
        xs, rows = [], []
        for s, (pt, w) in enumerate(c.systems(), start=1):
            pr = rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
            xs.append(pr.X)
            rows += [(r.system, r.rhs, r.init_relres, r.iterations, r.appended) for r in pr.log]
        outs.append((xs, rows, gb.batched_solves))
    assert outs[0][2] > 0
    assert outs[0][1] == outs[1][1]
    for xa, xb in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(xa, xb)


@pytest.mark.parametrize("cfg", ["T3c", "T2"])
def test_per_rhs_recycler_batched_matches_one_solve_path(rd, monkeypatch, cfg):
    """The per-RHS-only comparator's right-hand sides are always independent
    (basis.cpp:221-264), so its solves run batched; same BuildLog, solutions,
    stored directions and index lists as one solve at a time."""
    c = P.CONFIGS[cfg]
    g, lay = c.grid, c.layout()
    U0, X0 = _shared_seed(c, g, lay)
    runs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("ROMDOT_BATCH", mode)
        rec = rd.PerRhsRecycler(U0, X0)
        out = [rec.solve_system(rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s)
               for s, (pt, w) in enumerate(c.systems(), start=1)]
        runs[mode] = (out, rec.batched_solves, rec.cols, [rec.space(j) for j in range(lay.n_rhs)], rec.V)
    (a, n0, cols0, sp0, V0), (b, n1, cols1, sp1, V1) = runs["0"], runs["1"]
    assert n0 == 0 and n1 == lay.n_rhs * len(c.systems())
    assert cols0 == cols1 and sp0 == sp1
    for pa, pb in zip(a, b):
        for ra, rb in zip(pa.log, pb.log):
            assert (ra.system, ra.rhs, ra.appended) == (rb.system, rb.rhs, rb.appended)
            assert abs(ra.iterations - rb.iterations) <= 1
            assert rb.init_relres == pytest.approx(ra.init_relres, rel=1e-9, abs=1e-14)
        assert np.linalg.norm(pb.X - pa.X) <= 1e-8 * np.linalg.norm(pa.X)
    assert np.linalg.norm(V1 - V0) <= 1e-6 * np.linalg.norm(V0)
