"""ctypes wrapper of the CPU oracle (liboracle.so). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package never
does. See romdot_oracle.cpp's header for what it restates (file:line).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

c_long_p = C.POINTER(C.c_long)
c_int_p = C.POINTER(C.c_int)
c_double_p = C.POINTER(C.c_double)


def build(force: bool = False) -> str:
    so = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "romdot_oracle.cpp")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return so


def lib():
    global _LIB
    if _LIB is None:
        so = build()
        L = C.CDLL(so)
        vp = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        L.orc_op_grid.restype = vp
        L.orc_op_grid.argtypes = [C.c_int, C.c_int, c_long_p, C.c_double, C.c_double, vp, vp]
        L.orc_op_dense.restype = vp
        L.orc_op_dense.argtypes = [C.c_int, C.c_long, vp]
        L.orc_op_lam_max.restype = C.c_double
        L.orc_op_lam_max.argtypes = [vp]
        L.orc_op_apply.argtypes = [vp, vp, vp, C.c_long]
        L.orc_free_op.argtypes = [vp]
        L.orc_minres.argtypes = [vp, vp, C.c_double, C.c_long, vp, c_int_p, c_int_p, vp, C.c_long, c_long_p]
        L.orc_rs_from_raw.restype = vp
        L.orc_rs_from_raw.argtypes = [C.c_int, C.c_long, C.c_long, vp, vp]
        L.orc_rs_append.argtypes = [vp, vp, vp]
        L.orc_rs_cols.restype = C.c_long
        L.orc_rs_cols.argtypes = [vp]
        L.orc_rs_get.argtypes = [vp, vp, vp]
        L.orc_rs_initial_guess.argtypes = [vp, vp, vp, vp]
        L.orc_free_rs.argtypes = [vp]
        L.orc_recycled_solve.argtypes = [C.c_int, vp, vp, vp, C.c_double, C.c_long, C.c_double, vp, vp, vp,
                                         c_int_p, c_int_p, vp, C.c_long, c_long_p, c_double_p]
        L.orc_eigs.argtypes = [vp, C.c_long, C.c_double, vp, vp]
        L.orc_basis_from.restype = vp
        L.orc_basis_from.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, vp, vp, C.c_long]
        L.orc_free_basis.argtypes = [vp]
        L.orc_basis_cols.restype = C.c_long
        L.orc_basis_cols.argtypes = [vp]
        L.orc_basis_ku.restype = C.c_long
        L.orc_basis_ku.argtypes = [vp]
        L.orc_basis_get.argtypes = [vp, C.c_int, vp]
        L.orc_basis_markers.argtypes = [vp, vp]
        L.orc_basis_space.restype = C.c_long
        L.orc_basis_space.argtypes = [vp, C.c_long, vp]
        L.orc_basis_refresh.argtypes = [vp, vp]
        L.orc_basis_append.argtypes = [vp, vp, vp, C.c_int]
        L.orc_basis_solve_projected.argtypes = [vp, vp, vp, vp]
        L.orc_process_system.argtypes = [vp, vp, C.c_long, vp, vp, C.c_double, C.c_int, C.c_long, C.c_int,
                                         vp, vp, c_long_p, c_long_p]
        L.orc_initial_solutions.argtypes = [vp, C.c_long, vp, vp, C.c_double, C.c_int, vp, c_long_p]
        L.orc_per_rhs_create.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, vp, vp]
        L.orc_per_rhs_create.restype = vp
        L.orc_per_rhs_destroy.argtypes = [vp]
        L.orc_per_rhs_solve_system.argtypes = [vp, vp, C.c_long, vp, vp, C.c_double, C.c_int, C.c_long, C.c_int,
                                               vp, vp, c_long_p, c_long_p]
        L.orc_thin_qr.argtypes = [C.c_int, C.c_long, C.c_long, vp, vp, vp]
        L.orc_qrcp.argtypes = [C.c_int, C.c_long, C.c_long, vp, C.c_double, C.c_int, c_long_p, vp, vp, vp]
        L.orc_normal_stream.argtypes = [C.c_uint64, C.c_long, vp]
        L.orc_replay_rhs.argtypes = [vp, C.c_long, vp, vp, vp, vp, C.c_long, C.c_long, C.c_double, C.c_double,
                                     C.c_long, C.c_long, C.c_int, vp, vp, vp]
        _LIB = L
    return _LIB


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ConfigError(OracleError):
    pass


class SolverError(OracleError):
    pass


def _check(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        raise {2: ConfigError, 3: SolverError}.get(rc, OracleError)(rc, msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dt(dtype) -> int:
    return 1 if np.dtype(dtype) == np.complex128 else 0


def _f(a, dtype):
    return np.asfortranarray(a, dtype=dtype)


@dataclass
class Report:
    iterations: int
    converged: bool
    history: np.ndarray
    correction_norm: float = 0.0


class Operator:
    """Matrix-free operator (reference LinOp). Grid Schur operator or dense."""

    def __init__(self, handle, n, dtype):
        self.h = handle
        self.n = n
        self.dtype = np.dtype(dtype)

    @classmethod
    def grid(cls, grid, fields, dtype=np.float64):
        N = (C.c_long * 3)(*(list(grid.N) + [1] * (3 - grid.d)))
        D = np.ascontiguousarray(fields.D, dtype=np.float64)
        mu = np.ascontiguousarray(fields.mu, dtype=np.float64)
        h = lib().orc_op_grid(_dt(dtype), grid.d, N, grid.robin_face, float(fields.shift), _p(D), _p(mu))
        return cls(h, grid.n, dtype)

    @classmethod
    def dense(cls, A: np.ndarray):
        A = _f(A, A.dtype)
        h = lib().orc_op_dense(_dt(A.dtype), A.shape[0], _p(A))
        return cls(h, A.shape[0], A.dtype)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_free_op(self.h)
            self.h = None

    @property
    def lam_max(self) -> float:
        return lib().orc_op_lam_max(self.h)

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = _f(x, self.dtype)
        y = np.zeros_like(x)
        ncols = 1 if x.ndim == 1 else x.shape[1]
        _check(lib().orc_op_apply(self.h, _p(x), _p(y), ncols))
        return y

    def matrix(self) -> np.ndarray:
        return self.apply(np.eye(self.n, dtype=self.dtype))


def minres(op: Operator, b, tol, maxit):
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(op.n)
    its, conv, hl = C.c_int(), C.c_int(), C.c_long()
    hist = np.zeros(maxit + 2)
    _check(lib().orc_minres(op.h, _p(b), tol, maxit, _p(x), C.byref(its), C.byref(conv), _p(hist), hist.size,
                            C.byref(hl)))
    return x, Report(its.value, bool(conv.value), hist[: hl.value].copy())


class RecycleSpace:
    def __init__(self, W, AW):
        W = _f(W, W.dtype)
        AW = _f(AW, W.dtype)
        self.dtype = W.dtype
        self.n = W.shape[0]
        self.h = lib().orc_rs_from_raw(_dt(W.dtype), W.shape[0], W.shape[1], _p(W), _p(AW))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_free_rs(self.h)
            self.h = None

    def append(self, u, k) -> bool:
        u = np.ascontiguousarray(u, dtype=self.dtype)
        k = np.ascontiguousarray(k, dtype=self.dtype)
        return bool(lib().orc_rs_append(self.h, _p(u), _p(k)))

    @property
    def cols(self) -> int:
        return lib().orc_rs_cols(self.h)

    def UK(self):
        c = self.cols
        U = np.zeros((self.n, c), dtype=self.dtype, order="F")
        K = np.zeros_like(U)
        lib().orc_rs_get(self.h, _p(U), _p(K))
        return U, K

    def initial_guess(self, b):
        b = np.ascontiguousarray(b, dtype=self.dtype)
        z = np.zeros_like(b)
        r = np.zeros_like(b)
        lib().orc_rs_initial_guess(self.h, _p(b), _p(z), _p(r))
        return z, r


@dataclass
class RecycledResult:
    correction: np.ndarray
    new_direction: np.ndarray
    image: np.ndarray
    report: Report


MINRES, CG = 0, 1


def recycled_solve(method, op: Operator, rs: Optional[RecycleSpace], rhs, tol, maxit, rhs_scale=0.0):
    rhs = np.ascontiguousarray(rhs, dtype=op.dtype)
    corr, nd, im = (np.zeros(op.n, dtype=op.dtype) for _ in range(3))
    its, conv, hl, cn = C.c_int(), C.c_int(), C.c_long(), C.c_double()
    hist = np.zeros(maxit + 2)
    _check(lib().orc_recycled_solve(method, op.h, rs.h if rs is not None else None, _p(rhs), tol, maxit,
                                    rhs_scale, _p(corr), _p(nd), _p(im), C.byref(its), C.byref(conv), _p(hist),
                                    hist.size, C.byref(hl), C.byref(cn)))
    return RecycledResult(corr, nd, im, Report(its.value, bool(conv.value), hist[: hl.value].copy(), cn.value))


def recycled_minres(op, rs, rhs, tol, maxit, rhs_scale=0.0):
    return recycled_solve(MINRES, op, rs, rhs, tol, maxit, rhs_scale)


def recycled_cg(op, rs, rhs, tol, maxit, rhs_scale=0.0):
    return recycled_solve(CG, op, rs, rhs, tol, maxit, rhs_scale)


def smallest_eigenpairs(op: Operator, k: int, tol: float = 1e-8):
    lam = np.zeros(k)
    U = np.zeros((op.n, k), order="F")
    _check(lib().orc_eigs(op.h, k, tol, _p(lam), _p(U)))
    return lam, U


@dataclass
class LogRow:
    system: int
    rhs: int
    init_relres: float
    iterations: int
    appended: bool


@dataclass
class ProcessResult:
    X: np.ndarray
    log: List[LogRow]
    inner_iterations: int
    appends: int


class GlobalBasis:
    """GlobalBasis + PerRhsSpaces (basis.hpp:28-70)."""

    def __init__(self, U0, X0, cap: int = 0):
        dtype = np.result_type(U0.dtype, X0.dtype)
        U0 = _f(U0, dtype)
        X0 = _f(X0, dtype)
        self.dtype = np.dtype(dtype)
        self.n = U0.shape[0]
        self.nrhs = X0.shape[1]
        self.h = lib().orc_basis_from(_dt(dtype), self.n, U0.shape[1], X0.shape[1], _p(U0), _p(X0), cap)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_free_basis(self.h)
            self.h = None

    @property
    def cols(self) -> int:
        return lib().orc_basis_cols(self.h)

    @property
    def eig_block(self) -> int:
        return lib().orc_basis_ku(self.h)

    def _get(self, which, shape):
        out = np.zeros(shape, dtype=self.dtype, order="F")
        _check(lib().orc_basis_get(self.h, which, _p(out)))
        return out

    @property
    def V(self):
        return self._get(0, (self.n, self.cols))

    @property
    def K_img(self):
        return self._get(1, (self.n, self.cols))

    @property
    def R(self):
        return self._get(2, (self.cols, self.cols))

    @property
    def K_raw(self):
        return self._get(3, (self.n, self.cols))

    @property
    def markers(self):
        out = np.zeros(self.cols, dtype=np.uint8)
        lib().orc_basis_markers(self.h, _p(out))
        return out

    def space(self, j) -> List[int]:
        m = lib().orc_basis_space(self.h, j, None)
        out = np.zeros(max(m, 1), dtype=np.int32)
        lib().orc_basis_space(self.h, j, _p(out))
        return out[:m].tolist()

    def refresh(self, op: Operator):
        _check(lib().orc_basis_refresh(self.h, op.h))

    def append(self, y, z, marker=2) -> bool:
        y = np.ascontiguousarray(y, dtype=self.dtype)
        z = np.ascontiguousarray(z, dtype=self.dtype)
        return bool(lib().orc_basis_append(self.h, _p(y), _p(z), marker))

    def solve_projected(self, b):
        b = np.ascontiguousarray(b, dtype=self.dtype)
        x = np.zeros(self.n, dtype=self.dtype)
        c = np.zeros(self.cols, dtype=self.dtype)
        lib().orc_basis_solve_projected(self.h, _p(b), _p(x), _p(c))
        return x

    def projected_coordinates(self, b):
        b = np.ascontiguousarray(b, dtype=self.dtype)
        x = np.zeros(self.n, dtype=self.dtype)
        c = np.zeros(self.cols, dtype=self.dtype)
        lib().orc_basis_solve_projected(self.h, _p(b), _p(x), _p(c))
        return c


def process_system(gb: GlobalBasis, op: Operator, layout, tol, system_index, maxit=0, method=CG):
    nrhs = layout.n_rhs
    idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
    val = np.ascontiguousarray(layout.val, dtype=np.float64)
    X = np.zeros((gb.n, nrhs), dtype=gb.dtype, order="F")
    log = np.zeros((nrhs, 5))
    its, app = C.c_long(), C.c_long()
    _check(lib().orc_process_system(gb.h, op.h, nrhs, _p(idx), _p(val), tol, system_index, maxit, method, _p(X),
                                    _p(log), C.byref(its), C.byref(app)))
    rows = [LogRow(int(r[0]), int(r[1]), float(r[2]), int(r[3]), bool(r[4])) for r in log]
    return ProcessResult(X, rows, its.value, app.value)


class PerRhsRecycler:
    """BaselinePerRhsRecycler (basis.hpp:102-119, basis.cpp:209-266)."""

    def __init__(self, U0, X0):
        dt = np.result_type(U0.dtype, X0.dtype)
        U0 = np.asfortranarray(U0, dtype=dt)
        X0 = np.asfortranarray(X0, dtype=dt)
        self.dtype, self.n = dt, X0.shape[0]
        self.h = lib().orc_per_rhs_create(1 if dt == np.complex128 else 0, X0.shape[0], U0.shape[1], X0.shape[1],
                                          _p(U0), _p(X0))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_per_rhs_destroy(self.h)
            self.h = None

    def solve_system(self, op: Operator, layout, tol, system_index, maxit=0, method=CG):
        nrhs = layout.n_rhs
        idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
        val = np.ascontiguousarray(layout.val, dtype=np.float64)
        X = np.zeros((self.n, nrhs), dtype=self.dtype, order="F")
        log = np.zeros((nrhs, 5))
        its, app = C.c_long(), C.c_long()
        _check(lib().orc_per_rhs_solve_system(self.h, op.h, nrhs, _p(idx), _p(val), tol, system_index, maxit,
                                              method, _p(X), _p(log), C.byref(its), C.byref(app)))
        rows = [LogRow(int(r[0]), int(r[1]), float(r[2]), int(r[3]), bool(r[4])) for r in log]
        return ProcessResult(X, rows, its.value, app.value)


def initial_solutions(op: Operator, layout, tol, method=CG):
    idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
    val = np.ascontiguousarray(layout.val, dtype=np.float64)
    X0 = np.zeros((op.n, layout.n_rhs), dtype=op.dtype, order="F")
    tot = C.c_long()
    _check(lib().orc_initial_solutions(op.h, layout.n_rhs, _p(idx), _p(val), tol, method, _p(X0), C.byref(tot)))
    return X0, tot.value


def init_basis(op0: Operator, op0_real: Operator, layout, k_eig, tol, method=CG, cap=0, eig_tol=None):
    """basis.cpp:136-155: U0 from the omega=0 operator, X0 at 0.25 tol."""
    lam, U0 = smallest_eigenpairs(op0_real, k_eig, min(tol, 1e-8) if eig_tol is None else eig_tol)
    X0, its = initial_solutions(op0, layout, tol, method)
    gb = GlobalBasis(U0.astype(op0.dtype), X0, cap)
    return gb, X0, lam, U0


def thin_qr(A):
    A = _f(A, A.dtype)
    n, m = A.shape
    Q = np.zeros((n, m), dtype=A.dtype, order="F")
    R = np.zeros((m, m), dtype=A.dtype, order="F")
    _check(lib().orc_thin_qr(_dt(A.dtype), n, m, _p(A), _p(Q), _p(R)))
    return Q, R


def qrcp(A, tol=1e-10, normalize=True):
    """normalize=True: unit-norm columns first (basis compression, App. A9)."""
    A = _f(A, A.dtype)
    n, m = A.shape
    rank = C.c_long()
    perm = np.zeros(m, dtype=np.int64)
    rdiag = np.zeros(min(n, m))
    Q = np.zeros((n, m), dtype=A.dtype, order="F")
    _check(lib().orc_qrcp(_dt(A.dtype), n, m, _p(A), tol, int(normalize), C.byref(rank), _p(perm), _p(rdiag), _p(Q)))
    return rank.value, perm, rdiag, Q[:, : rank.value].copy()


def normal_stream(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count)
    lib().orc_normal_stream(seed, count, _p(out))
    return out


@dataclass
class ReplayResult:
    """One process_system RHS replayed from a recorded state (replay_rhs)."""
    init_relres: float
    iterations: int
    appended: bool
    rho_over_znorm: float
    converged: bool
    room: bool
    X: np.ndarray
    y: Optional[np.ndarray]
    times: dict


def replay_rhs(op: Operator, V, K_img, R, space, bidx: int, bval: float, tol: float, cap: int = 0, maxit: int = 0,
               method=CG, want_y: bool = False) -> ReplayResult:
    """The loop body of process_system (basis.cpp:168-205) for one RHS, run on
    a recorded basis state (V, K_img: n x r Fortran views, R: r x r) without
    copying it: global check, recycle space from_raw(V[:, space], A V[:, space]),
    recycled CG/COCG at 0.25 tol, X_j = correction + solve_projected(b_j), and
    the append decision (not applied). Host-core wall times per phase."""
    n, r = V.shape
    for a in (V, K_img):
        if a.dtype != op.dtype or not a.flags.f_contiguous or a.shape != (n, r):
            raise ValueError("replay_rhs: V / K_img must be Fortran (n, r) arrays of the operator dtype")
    Rf = _f(R, op.dtype)
    sp = np.ascontiguousarray(space, dtype=np.int32)
    X = np.zeros(n, dtype=op.dtype)
    y = np.zeros(n, dtype=op.dtype) if want_y else None
    info = np.zeros(12)
    _check(lib().orc_replay_rhs(op.h, r, _p(V), _p(K_img), _p(Rf), _p(sp), sp.size, int(bidx), float(bval), tol,
                                maxit, cap, method, _p(X), _p(y) if y is not None else None, _p(info)))
    keys = ["check", "space", "solve", "projected", "append", "total"]
    return ReplayResult(float(info[0]), int(info[1]), bool(info[2]), float(info[3]), bool(info[4]), bool(info[11]),
                        X, y, dict(zip(keys, map(float, info[5:11]))))
