"""Device ReducedModel (reference src/rom.cpp:9-67,
tests/test_rom.cpp, acceptance C3) against numpy on the same inputs.

* E_r, A_r = sym(V^T A V), Psi_r = C_r^T A_r^-1 B_r and the support-row
  Jacobian, real and complex (bilinear projections), <= 1e-10 relative;
* the rank-deficiency error of the constructor (rom.cpp:12-14);
* interpolation: the ROM of a device-built, device-compressed basis matches
  the full-order transfer at the build's own parameters (acceptance.cpp
  C3 `:252-274`, tolerance 1e-5 there).
"""
import numpy as np
import pytest

import oracle as orc
from paper_1602_00138_b200 import problem as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_1602_00138_b200 import romdot
    return romdot


def _orth(n, r, cplx, seed):
    g = np.random.default_rng(seed)
    A = g.standard_normal((n, r))
    if cplx:
        A = A + 1j * g.standard_normal((n, r))
    return np.linalg.qr(A)[0]


def _supports(n, npar, seed):
    g = np.random.default_rng(seed)
    out = []
    for k in range(npar):
        m = int(g.integers(1, n // 4))
        ix = np.sort(g.choice(n, size=m, replace=False))
        out.append((ix, g.uniform(0.1, 1.0, m)))
    out.append((np.zeros(0, dtype=np.int64), np.zeros(0)))  # empty support -> zero column (rom.cpp:52-55)
    return out


def _expected(V, A, B, C, supports, scale):
    Ar = V.T @ (A @ V)
    Ar = 0.5 * (Ar + Ar.T)
    Y = np.linalg.solve(Ar, V.T @ B)
    Z = np.linalg.solve(Ar, V.T @ C)
    Psi = (V.T @ C).T @ Y
    WY, WZ = V @ Y, V @ Z
    J = np.zeros((C.shape[1] * B.shape[1], len(supports)), dtype=np.result_type(V, A))
    for k, (ix, w) in enumerate(supports):
        M = (WZ[ix] * w[:, None]).T @ WY[ix]  # n_det x n_src (rom.cpp:60)
        J[:, k] = scale * M.ravel(order="F")  # Eigen column-major vec (rom.cpp:61)
    return Ar, Psi, J


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", ["T3", "T3c", "T2c"])
def test_rom_matches_numpy(rd, name):
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    pt, w = c.systems()[-1]
    f = c.fields(pt, w)
    A = orc.Operator.grid(g, f, c.dtype).matrix()
    Bc = lay.dense(g.n)
    B, C = Bc[:, : lay.n_src], Bc[:, lay.n_src:]
    V = _orth(g.n, 24, c.complex, 7)
    rom = rd.ReducedModel(V)
    op = rd.SchurOperator(g, f, c.dtype)
    sup = _supports(g.n, 3, 11)
    scale = -g.h ** 2
    Ar, Psi, J = _expected(V, A, B, C, sup, scale)
    assert rom.order() == 24
    assert _rel(rom.E_r, V.T @ V) <= 1e-13
    assert _rel(rom.reduced_system(op), Ar) <= 1e-12
    assert _rel(rom.transfer(op, lay), Psi) <= 1e-10
    Jd = rom.jacobian(op, lay, sup, scale)
    assert Jd.shape == J.shape
    assert _rel(Jd, J) <= 1e-10
    assert np.all(Jd[:, -1] == 0)


def test_rom_rank_deficient_basis_is_solver_error(rd):
    c = P.CONFIGS["T3"]
    V = _orth(c.grid.n, 6, False, 3)
    V = np.concatenate([V, V[:, :1]], axis=1)
    with pytest.raises(rd.SolverError, match="rank deficient"):
        rd.ReducedModel(V)


def test_rom_real_model_rejects_complex_operator(rd):
    c = P.CONFIGS["T3c"]
    rom = rd.ReducedModel(_orth(c.grid.n, 5, False, 2))
    op = rd.SchurOperator(c.grid, c.fields(1, 0.1), np.complex128)
    with pytest.raises(rd.ConfigError):
        rom.transfer(op, c.layout())


@pytest.mark.parametrize("name", ["T3", "T3c"])
def test_rom_of_compressed_device_basis_interpolates_fom(rd, name):
    """acceptance.cpp C3 (:252-274): ROM transfer at the basis parameters
    equals the FOM transfer (reference tolerance 1e-5)."""
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    op0r = rd.SchurOperator(g, c.fields(0), np.float64)
    op0 = rd.SchurOperator(g, c.fields(0), c.dtype)
    gb, _, _, _ = rd.init_basis(op0, op0r, lay, c.k, c.tol, c.cap)
    for s, (pt, w) in enumerate(c.systems(), start=1):
        rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s, want_X=False)
    rank, _, _ = gb.compress(1e-10)
    assert rank == gb.cols
    from paper_1602_00138_b200 import romdot as R
    vptr = R.load_library().rd_basis_device_ptr(gb.h, 0)
    rom = rd.ReducedModel(vptr, dtype=c.dtype, where=rd.DEVICE, n=g.n, r=rank)
    Bc = lay.dense(g.n)
    B, C = Bc[:, : lay.n_src], Bc[:, lay.n_src:]
    for pt, w in c.systems():
        f = c.fields(pt, w)
        A = orc.Operator.grid(g, f, c.dtype).matrix()
        fom = C.T @ np.linalg.solve(A, B)
        psi = rom.transfer(rd.SchurOperator(g, f, c.dtype), lay)
        assert _rel(psi, fom) <= 1e-5, (pt, w, _rel(psi, fom))
    del rom


# ---------------------------------------------------------------------------
# Full-order model and batched X0 solves

@pytest.mark.parametrize("name", ["T3", "T3c", "T2c"])
def test_fom_transfer_and_jacobian_match_dense(rd, name):
    """fom_transfer / fom_jacobian (rom.cpp:86-129) by batched CG/COCG vs
    dense solves. Psi samples X at far-field detector nodes (~1e-3 of ||x||),
    so the solves run at 1e-12 for a 1e-8 bound on the outputs."""
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    pt, w = c.systems()[-1]
    f = c.fields(pt, w)
    A = orc.Operator.grid(g, f, c.dtype).matrix()
    Bc = lay.dense(g.n)
    B, C = Bc[:, : lay.n_src], Bc[:, lay.n_src:]
    X = np.linalg.solve(A, B)
    Z = np.linalg.solve(A, C)
    op = rd.SchurOperator(g, f, c.dtype)
    psi, its = rd.fom_transfer(op, lay, 1e-12)
    assert its > 0
    assert _rel(psi, C.T @ X) <= 1e-8
    sup = _supports(g.n, 4, 5)
    scale = -g.h ** 2
    J = np.zeros((lay.n_det * lay.n_src, len(sup)), dtype=X.dtype)
    for k, (ix, wv) in enumerate(sup):
        M = (Z[ix] * wv[:, None]).T @ X[ix]  # jacobian_from_solutions, rom.cpp:118-124
        J[:, k] = scale * M.ravel(order="F")
    Jd = rd.fom_jacobian(op, lay, sup, scale, 1e-12)
    assert _rel(Jd[:, :-1], J[:, :-1]) <= 1e-8
    assert np.all(Jd[:, -1] == 0)


@pytest.mark.parametrize("name", ["T2", "T3c"])
def test_batched_initial_solutions_match_oracle(rd, name):
    """init_basis X0 (basis.cpp:141-149): the batched device solves meet the
    0.25 tol residual per column and agree with the CPU checker's solutions."""
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    f0 = c.fields(0)
    X0, its = rd.initial_solutions(rd.SchurOperator(g, f0, c.dtype), lay, c.tol)
    Xo, its_o = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    A = orc.Operator.grid(g, f0, c.dtype).matrix()
    B = lay.dense(g.n, c.dtype)
    res = np.linalg.norm(A @ X0 - B, axis=0) / np.linalg.norm(B, axis=0)
    assert res.max() <= 0.25 * c.tol * 1.01
    assert abs(its - its_o) <= 2 * lay.n_rhs
    err = np.linalg.norm(X0 - Xo, axis=0) / np.linalg.norm(Xo, axis=0)
    assert err.max() <= 1e-6


def test_fom_errors(rd):
    c = P.CONFIGS["T3c"]
    lay = c.layout()
    op = rd.SchurOperator(c.grid, c.fields(1, 0.2), np.complex128)
    opr = rd.SchurOperator(c.grid, c.fields(1, 0.0), np.float64)
    with pytest.raises(rd.ConfigError):
        bad = P.Layout(idx=np.array(list(lay.idx[:-1]) + [c.grid.n]), val=lay.val, n_src=lay.n_src, n_det=lay.n_det)
        rd.fom_transfer(op, bad, 1e-10)
    # real dtype with a complex shift is a configuration error
    opr.set_fields(c.fields(1, 0.2))
    with pytest.raises(rd.ConfigError):
        rd.fom_transfer(opr, lay, 1e-10)


# ---------------------------------------------------------------------------
# Offline seed cache and basis files

def test_offline_seed_cached_by_config_hash(rd, tmp_path):  # test_harness.cpp:202-217
    from paper_1602_00138_b200 import offline as O
    c = P.CONFIGS["T3"]
    d = str(tmp_path / "offline")
    assert not O.offline_seed(c, d)   # computed
    assert O.offline_seed(c, d)       # cached
    m = O.read_manifest(d + "/offline_manifest.txt")
    m["hash"] = "0000000000000000"    # tampering forces a recompute
    O.write_manifest(d + "/offline_manifest.txt", m)
    assert not O.offline_seed(c, d)
    U0, X0 = O.load_seed(d)
    assert U0.shape == (c.grid.n, c.k) and X0.shape == (c.grid.n, c.layout().n_rhs)
    mk = rd.romb_read(d + "/u0.romb")[1]
    assert np.all(mk == O.COL_EIGENVECTOR)


@pytest.mark.parametrize("name", ["T3", "T3c"])
def test_build_from_cached_seed_and_basis_file(rd, tmp_path, name):
    """init_basis_from on the cached seed (basis.cpp:114-134) reproduces the
    freshly seeded build bit for bit; write_basis of the device basis reads
    back bit-exactly with its markers."""
    from paper_1602_00138_b200 import offline as O
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    d = str(tmp_path / "seed")
    O.offline_seed(c, d)
    U0, X0 = O.load_seed(d)

    def build(U0, X0):
        gb = rd.GlobalBasis(U0.astype(c.dtype), X0, c.cap)
        logs = []
        for s, (pt, w) in enumerate(c.systems(), start=1):
            pr = rd.process_system(gb, rd.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s, want_X=False)
            logs += [(r.init_relres, r.iterations, r.appended) for r in pr.log]
        return gb, logs

    op0r = rd.SchurOperator(g, c.fields(0), np.float64)
    op0 = rd.SchurOperator(g, c.fields(0), c.dtype)
    _, U0f = rd.smallest_eigenpairs(op0r, c.k, min(c.tol, 1e-8))
    X0f, _ = rd.initial_solutions(op0, lay, c.tol)
    gb1, log1 = build(U0, X0)
    gb2, log2 = build(U0f, X0f)
    assert log1 == log2
    path = str(tmp_path / "basis.romb")
    gb1.save(path)
    V, mk = rd.romb_read(path)
    assert V.tobytes(order="F") == gb1.V.tobytes(order="F")
    assert np.array_equal(mk, gb1.markers[: gb1.cols])
