"""Python mirror of the reference's basis-builder API over the C ABI
(include/romdot_b200.h), backed by libromdot_b200.so (CUDA, sm_100a).

Names and semantics follow the reference (proj/include/romdot/{grid,krylov,
basis}.hpp): ``SchurOperator.apply``, ``RecycleSpace``, ``recycled_cg`` (the
CG/COCG counterpart of ``recycled_minres``), ``GlobalBasis`` with
``refresh/append/solve_projected/projected_coordinates/V/K_img/R/markers``,
``init_basis`` / ``init_basis_from`` and ``process_system``. Errors map to
``ConfigError`` / ``SolverError`` like the reference's exception taxonomy
(include/romdot/types.hpp:20-30).

There is no CPU fallback: importing this module without the built library, or
calling it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import problem as P

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libromdot_b200.so")

EXPORTS = [
    "rd_ctx_create", "rd_ctx_destroy", "rd_last_error", "rd_ctx_sync", "rd_ctx_mark", "rd_ctx_elapsed_ms",
    "rd_ctx_launches", "rd_ctx_set_solver", "rd_ctx_get_solver", "rd_ctx_stream", "rd_ctx_profile", "rd_ctx_prof_get", "rd_op_create", "rd_op_destroy", "rd_op_set_fields", "rd_op_apply",
    "rd_op_lam_max", "rd_recycled_solve", "rd_recycle_space_from_raw", "rd_initial_solutions",
    "rd_smallest_eigenpairs", "rd_basis_create", "rd_basis_destroy", "rd_basis_cols", "rd_basis_factored", "rd_basis_eig_block", "rd_basis_batched_solves",
    "rd_basis_get", "rd_basis_device_ptr", "rd_basis_markers", "rd_basis_space", "rd_basis_refresh",
    "rd_basis_append", "rd_basis_solve_projected", "rd_process_system", "rd_rrqr", "rd_bench_projection",
    "rd_bench_stencil", "rd_residual_norms", "rd_basis_compress", "rd_rom_create", "rd_rom_destroy",
    "rd_rom_order", "rd_rom_E", "rd_rom_reduced_system", "rd_rom_transfer", "rd_rom_jacobian",
    "rd_fom_transfer", "rd_fom_jacobian", "rd_per_rhs_create", "rd_per_rhs_solve_system",
    "rd_romb_write", "rd_romb_info", "rd_romb_read", "rd_basis_save", "rd_bench_gram", "rd_basis_set_rhs_hook", "rd_bench_gemm", "rd_ctx_fused_check",
]


class RomdotError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ConfigError(RomdotError):
    pass


class SolverError(RomdotError):
    pass


class CudaError(RomdotError):
    pass


class IoError(RomdotError):
    """IoError (types.hpp:28-30): basis / manifest files."""


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("correction_norm", C.c_double),
                ("final_relres", C.c_double)]


_LIB = None

# int (*)(void* user, int system_index, long rhs): rd_basis_set_rhs_hook
RHS_HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_long)


def load_library(path: Optional[str] = None):
    """Load libromdot_b200.so (raises if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    so = path or _SO
    if not os.path.exists(so):
        raise ImportError(f"{so} not built: run `python -m paper_1602_00138_b200.build` (no CPU fallback)")
    L = C.CDLL(so)
    vp, lp, ip, dp = C.c_void_p, C.POINTER(C.c_long), C.POINTER(C.c_int), C.POINTER(C.c_double)
    L.rd_last_error.restype = C.c_char_p
    L.rd_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.rd_ctx_destroy.argtypes = [vp]
    L.rd_ctx_sync.argtypes = [vp]
    L.rd_ctx_mark.argtypes = [vp]
    L.rd_ctx_elapsed_ms.argtypes = [vp]
    L.rd_ctx_elapsed_ms.restype = C.c_double
    L.rd_ctx_launches.argtypes = [vp]
    L.rd_ctx_launches.restype = C.c_long
    L.rd_ctx_set_solver.argtypes = [vp, C.c_int]
    L.rd_ctx_get_solver.argtypes = [vp]
    L.rd_ctx_fused_check.argtypes = [vp, lp, lp]
    L.rd_ctx_fused_check.restype = None
    L.rd_ctx_stream.argtypes = [vp]
    L.rd_ctx_stream.restype = vp
    L.rd_ctx_profile.argtypes = [vp, C.c_int]
    L.rd_ctx_profile.restype = None
    L.rd_ctx_prof_get.argtypes = [vp, C.c_int, dp, dp, lp]
    L.rd_op_create.argtypes = [vp, C.c_int, lp, C.c_double, C.POINTER(vp)]
    L.rd_op_destroy.argtypes = [vp]
    L.rd_op_set_fields.argtypes = [vp, vp, vp, C.c_double, C.c_int]
    L.rd_op_apply.argtypes = [vp, C.c_int, vp, vp, C.c_long, C.c_int]
    L.rd_op_lam_max.argtypes = [vp]
    L.rd_op_lam_max.restype = C.c_double
    L.rd_recycled_solve.argtypes = [vp, C.c_int, vp, vp, C.c_long, vp, C.c_double, C.c_long, C.c_double, vp, vp, vp,
                                    C.POINTER(_Report), vp, C.c_long, C.c_int]
    L.rd_recycle_space_from_raw.argtypes = [vp, C.c_int, C.c_long, C.c_long, vp, vp, vp, vp, C.c_int]
    L.rd_initial_solutions.argtypes = [vp, C.c_int, C.c_long, vp, vp, C.c_double, vp, C.c_int, lp]
    L.rd_smallest_eigenpairs.argtypes = [vp, C.c_long, C.c_double, vp, vp, C.c_int]
    L.rd_basis_create.argtypes = [vp, C.c_int, C.c_long, C.c_long, C.c_long, vp, vp, C.c_long, C.c_int,
                                  C.POINTER(vp)]
    L.rd_basis_destroy.argtypes = [vp]
    L.rd_basis_cols.argtypes = [vp]
    L.rd_basis_cols.restype = C.c_long
    L.rd_basis_factored.argtypes = [vp]
    L.rd_basis_factored.restype = C.c_int
    L.rd_basis_eig_block.argtypes = [vp]
    L.rd_basis_eig_block.restype = C.c_long
    L.rd_basis_batched_solves.argtypes = [vp]
    L.rd_basis_batched_solves.restype = C.c_long
    L.rd_basis_get.argtypes = [vp, C.c_int, vp]
    L.rd_basis_device_ptr.argtypes = [vp, C.c_int]
    L.rd_basis_device_ptr.restype = vp
    L.rd_basis_markers.argtypes = [vp, vp]
    L.rd_basis_space.argtypes = [vp, C.c_long, vp]
    L.rd_basis_space.restype = C.c_long
    L.rd_basis_refresh.argtypes = [vp, vp]
    L.rd_basis_append.argtypes = [vp, vp, vp, C.c_int, C.c_int, ip]
    L.rd_basis_solve_projected.argtypes = [vp, vp, vp, vp, C.c_int]
    L.rd_process_system.argtypes = [vp, vp, C.c_long, vp, vp, C.c_double, C.c_int, C.c_long, vp, C.c_int, vp, lp,
                                    lp]
    L.rd_rrqr.argtypes = [vp, C.c_int, C.c_long, C.c_long, vp, C.c_double, C.c_int, lp, vp, vp, vp, C.c_int]
    L.rd_bench_projection.argtypes = [vp, C.c_int, C.c_long, C.c_long, C.c_int, vp]
    L.rd_bench_stencil.argtypes = [vp, C.c_int, C.c_long, C.c_int, vp]
    L.rd_bench_gram.argtypes = [vp, C.c_int, C.c_long, C.c_long, C.c_long, C.c_int, C.c_int, vp]
    L.rd_bench_gemm.argtypes = [vp, C.c_int, C.c_long, C.c_long, C.c_long, C.c_int, C.c_int, vp]
    L.rd_basis_compress.argtypes = [vp, C.c_double, C.c_int, lp, vp, vp]
    L.rd_residual_norms.argtypes = [vp, C.c_int, C.c_long, vp, vp, vp, C.c_int, vp]
    L.rd_romb_write.argtypes = [C.c_char_p, C.c_int, C.c_long, C.c_long, vp, vp, C.c_int, vp]
    L.rd_romb_info.argtypes = [C.c_char_p, C.POINTER(C.c_int), lp, lp]
    L.rd_romb_read.argtypes = [C.c_char_p, C.c_int, C.c_long, C.c_long, vp, vp, C.c_int, vp]
    L.rd_basis_save.argtypes = [vp, C.c_char_p]
    L.rd_per_rhs_create.argtypes = [vp, C.c_int, C.c_long, C.c_long, C.c_long, vp, vp, C.c_int, C.POINTER(vp)]
    L.rd_per_rhs_solve_system.argtypes = [vp, vp, C.c_long, vp, vp, C.c_double, C.c_int, C.c_long, vp, C.c_int, vp,
                                          lp, lp]
    L.rd_fom_transfer.argtypes = [vp, C.c_int, C.c_long, vp, vp, C.c_long, vp, vp, C.c_double, vp, C.c_int, lp]
    L.rd_fom_jacobian.argtypes = [vp, C.c_int, C.c_long, vp, vp, C.c_long, vp, vp, C.c_long, vp, vp, vp, C.c_double,
                                  C.c_double, vp, C.c_int]
    L.rd_basis_set_rhs_hook.argtypes = [vp, RHS_HOOK, vp]
    L.rd_rom_create.argtypes = [vp, C.c_int, C.c_long, C.c_long, vp, C.c_int, C.POINTER(vp)]
    L.rd_rom_destroy.argtypes = [vp]
    L.rd_rom_order.argtypes = [vp]
    L.rd_rom_order.restype = C.c_long
    L.rd_rom_E.argtypes = [vp, vp, C.c_int]
    L.rd_rom_reduced_system.argtypes = [vp, vp, vp, C.c_int]
    L.rd_rom_transfer.argtypes = [vp, vp, C.c_long, vp, vp, C.c_long, vp, vp, vp, C.c_int]
    L.rd_rom_jacobian.argtypes = [vp, vp, C.c_long, vp, vp, C.c_long, vp, vp, C.c_long, vp, vp, vp, C.c_double,
                                  vp, C.c_int]
    _LIB = L
    return L


def _release(fn: str, h) -> None:
    """Destructor helper: free a handle unless the interpreter is shutting
    down (module globals already cleared)."""
    try:
        lib = globals().get("_LIB")
        if lib is not None and h:
            getattr(lib, fn)(h)
    except Exception:  # interpreter teardown
        pass


def _check(rc):
    if rc != 0:
        msg = load_library().rd_last_error().decode()
        raise {2: ConfigError, 3: SolverError, 4: IoError, 5: CudaError}.get(rc, RomdotError)(rc, msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dt(dtype) -> int:
    return 1 if np.dtype(dtype) == np.complex128 else 0


def _f(a, dtype):
    return np.asfortranarray(a, dtype=dtype)


HOST, DEVICE = 0, 1


class Context:
    """Device, stream and reduction workspace (one per host thread)."""

    def __init__(self, device: int = 0):
        L = load_library()
        h = C.c_void_p()
        _check(L.rd_ctx_create(device, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _release("rd_ctx_destroy", self.h)
            except Exception:
                pass
            self.h = None

    def sync(self):
        _check(load_library().rd_ctx_sync(self.h))

    def mark(self):
        _check(load_library().rd_ctx_mark(self.h))

    def elapsed_ms(self) -> float:
        return load_library().rd_ctx_elapsed_ms(self.h)

    @property
    def launches(self) -> int:
        return load_library().rd_ctx_launches(self.h)

    def profile(self, enable: bool = True):
        load_library().rd_ctx_profile(self.h, int(enable))

    CG, MINRES = 0, 1

    def set_solver(self, solver: int):
        """0 = recycled CG / COCG (default, the hot path); 1 = the reference's
        recycled MINRES (krylov.cpp:17-98, 147-179; real operators, parity path)."""
        _check(load_library().rd_ctx_set_solver(self.h, int(solver)))

    @property
    def solver(self) -> int:
        return load_library().rd_ctx_get_solver(self.h)

    PROF_CLASSES = ("cg_stencil_dots", "ts_T", "ts_NT", "cg_update", "cg_fused", "bcg_defl_step", "bcg_defl_slot_steps")

    def prof(self):
        """{class: (ms_total, algorithmic_bytes_total, samples)} of the sampled launches."""
        out = {}
        for i, name in enumerate(self.PROF_CLASSES):
            ms, by, ns = C.c_double(), C.c_double(), C.c_long()
            load_library().rd_ctx_prof_get(self.h, i, C.byref(ms), C.byref(by), C.byref(ns))
            out[name] = (ms.value, by.value, ns.value)
        return out

    def fused_check(self):
        """(fused launches checked, stale halo reads) under ROMDOT_FUSED_CHECK=1."""
        a, b = C.c_long(), C.c_long()
        load_library().rd_ctx_fused_check(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    @property
    def stream(self) -> int:
        return load_library().rd_ctx_stream(self.h)


_DEFAULT_CTX: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Context(0)
    return _DEFAULT_CTX


class SchurOperator:
    """Device Schur operator A~(p) (grid.hpp:100-114): 5/7-point variable-D
    stencil with the eliminated Robin layers, coefficient fields per system."""

    def __init__(self, grid: P.GridSpec, fields: Optional[P.Fields] = None, dtype=np.float64,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.grid = grid
        self.n = grid.n
        self.dtype = np.dtype(dtype)
        N = (C.c_long * 3)(*(list(grid.N) + [1] * (3 - grid.d)))
        h = C.c_void_p()
        _check(load_library().rd_op_create(self.ctx.h, grid.d, N, grid.robin_face, C.byref(h)))
        self.h = h
        if fields is not None:
            self.set_fields(fields)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _release("rd_op_destroy", self.h)
            except Exception:
                pass
            self.h = None

    def set_fields(self, fields: P.Fields, where: int = HOST, D_ptr=None, mu_ptr=None):
        if where == DEVICE:
            _check(load_library().rd_op_set_fields(self.h, D_ptr, mu_ptr, float(fields.shift), DEVICE))
        else:
            D = np.ascontiguousarray(fields.D, dtype=np.float64)
            mu = np.ascontiguousarray(fields.mu, dtype=np.float64)
            _check(load_library().rd_op_set_fields(self.h, _p(D), _p(mu), float(fields.shift), HOST))
        self.fields = fields

    @property
    def lam_max(self) -> float:
        return load_library().rd_op_lam_max(self.h)

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = _f(x, self.dtype)
        y = np.zeros_like(x)
        ncols = 1 if x.ndim == 1 else x.shape[1]
        _check(load_library().rd_op_apply(self.h, _dt(self.dtype), _p(x), _p(y), ncols, HOST))
        return y


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    rel_residual_history: np.ndarray
    correction_norm: float
    final_relres: float


@dataclass
class RecycledResult:
    correction: np.ndarray
    new_direction: np.ndarray
    image: np.ndarray
    report: SolveReport


def recycled_cg(op: SchurOperator, U: Optional[np.ndarray], K: Optional[np.ndarray], rhs, tol, maxit,
                rhs_scale: float = 0.0) -> RecycledResult:
    """Deflated CG / COCG on the correction equation (krylov.hpp:53-58 semantics)."""
    dt = op.dtype
    rhs = np.ascontiguousarray(rhs, dtype=dt)
    c = 0 if U is None else U.shape[1]
    Uf = _f(U, dt) if c else None
    Kf = _f(K, dt) if c else None
    g, y, im = (np.zeros(op.n, dtype=dt) for _ in range(3))
    rep = _Report()
    hist = np.zeros(min(maxit + 2, 1 << 16))
    _check(load_library().rd_recycled_solve(op.h, _dt(dt), _p(Uf), _p(Kf), c, _p(rhs), tol, maxit, rhs_scale,
                                            _p(g), _p(y), _p(im), C.byref(rep), _p(hist), hist.size, HOST))
    m = min(rep.iterations + 1, hist.size)
    return RecycledResult(g, y, im, SolveReport(rep.iterations, bool(rep.converged), hist[:m].copy(),
                                                rep.correction_norm, rep.final_relres))


def recycled_minres(op: SchurOperator, U: Optional[np.ndarray], K: Optional[np.ndarray], rhs, tol, maxit,
                    rhs_scale: float = 0.0) -> RecycledResult:
    """The reference's own inner solver on the device (krylov.cpp:147-179, real
    operators): `recycled_cg` with the context switched to MINRES for the call."""
    prev = op.ctx.solver
    op.ctx.set_solver(Context.MINRES)
    try:
        return recycled_cg(op, U, K, rhs, tol, maxit, rhs_scale)
    finally:
        op.ctx.set_solver(prev)


def recycle_space_from_raw(W: np.ndarray, AW: np.ndarray, ctx: Optional[Context] = None):
    """RecycleSpace::from_raw (krylov.cpp:106-115) on the device: returns (U, K)."""
    ctx = ctx or default_context()
    dt = W.dtype
    W = _f(W, dt)
    AW = _f(AW, dt)
    U = np.zeros_like(W)
    K = np.zeros_like(W)
    _check(load_library().rd_recycle_space_from_raw(ctx.h, _dt(dt), W.shape[0], W.shape[1], _p(W), _p(AW), _p(U),
                                                    _p(K), HOST))
    return U, K


def initial_solutions(op: SchurOperator, layout: P.Layout, tol: float):
    """X0 columns of init_basis (basis.cpp:141-149), CG/COCG at 0.25 tol."""
    idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
    val = np.ascontiguousarray(layout.val, dtype=np.float64)
    X0 = np.zeros((op.n, layout.n_rhs), dtype=op.dtype, order="F")
    tot = C.c_long()
    _check(load_library().rd_initial_solutions(op.h, _dt(op.dtype), layout.n_rhs, _p(idx), _p(val), tol, _p(X0),
                                               HOST, C.byref(tot)))
    return X0, tot.value


def smallest_eigenpairs(op: SchurOperator, k: int, tol: float = 1e-8):
    lam = np.zeros(k)
    U = np.zeros((op.n, k), order="F")
    _check(load_library().rd_smallest_eigenpairs(op.h, k, tol, _p(lam), _p(U), HOST))
    return lam, U


@dataclass
class BuildLogRow:
    system: int
    rhs: int
    init_relres: float
    iterations: int
    appended: bool


@dataclass
class ProcessResult:
    X: Optional[np.ndarray]
    log: List[BuildLogRow]
    inner_iterations: int
    appends: int


class GlobalBasis:
    """Device GlobalBasis + PerRhsSpaces (basis.hpp:28-70)."""

    def __init__(self, U0: np.ndarray, X0: np.ndarray, cap: int = 0, ctx: Optional[Context] = None,
                 dtype=None):
        self.ctx = ctx or default_context()
        dt = np.dtype(dtype) if dtype is not None else np.result_type(U0.dtype, X0.dtype)
        U0 = _f(U0, dt)
        X0 = _f(X0, dt)
        self.dtype = dt
        self.n = X0.shape[0]
        self.nrhs = X0.shape[1]
        h = C.c_void_p()
        _check(load_library().rd_basis_create(self.ctx.h, _dt(dt), self.n, U0.shape[1], X0.shape[1], _p(U0), _p(X0),
                                              cap, HOST, C.byref(h)))
        self.h = h

    @classmethod
    def from_device(cls, U0_ptr: int, X0_ptr: int, n: int, ku: int, nrhs: int, dtype, cap: int = 0,
                    ctx: Optional[Context] = None) -> "GlobalBasis":
        """init_basis_from (basis.cpp:114-134) on device-resident U0 (n x ku) and
        X0 (n x nrhs), column-major, already in the basis dtype (no host copy)."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.dtype = np.dtype(dtype)
        self.n, self.nrhs = n, nrhs
        h = C.c_void_p()
        _check(load_library().rd_basis_create(self.ctx.h, _dt(self.dtype), n, ku, nrhs, C.c_void_p(U0_ptr),
                                              C.c_void_p(X0_ptr), cap, DEVICE, C.byref(h)))
        self.h = h
        return self

    def destroy(self):
        """Free the device buffers now (instead of at garbage collection)."""
        if getattr(self, "h", None):
            load_library().rd_basis_destroy(self.h)
            self.h = None

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _release("rd_basis_destroy", self.h)
            except Exception:
                pass
            self.h = None

    @property
    def cols(self) -> int:
        return load_library().rd_basis_cols(self.h)

    @property
    def eig_block(self) -> int:
        return load_library().rd_basis_eig_block(self.h)

    @property
    def batched_solves(self) -> int:
        """Correction solves that ran in the batched iteration (independent RHS after the cap)."""
        return load_library().rd_basis_batched_solves(self.h)

    def _get(self, which, shape):
        out = np.zeros(shape, dtype=self.dtype, order="F")
        _check(load_library().rd_basis_get(self.h, which, _p(out)))
        return out

    @property
    def V(self):
        return self._get(0, (self.n, self.cols))

    @property
    def factored(self) -> bool:
        """True once refresh has built the image factor A V = K_img R."""
        return bool(load_library().rd_basis_factored(self.h))

    @property
    def K_img(self):
        """Orthonormal image basis; empty (n x 0) before the first refresh, like the reference."""
        if not self.factored:
            return np.zeros((self.n, 0), dtype=self.dtype, order="F")
        return self._get(1, (self.n, self.cols))

    @property
    def R(self):
        if not self.factored:
            return np.zeros((0, 0), dtype=self.dtype, order="F")
        return self._get(2, (self.cols, self.cols))

    @property
    def W(self):
        if not self.factored:
            return np.zeros((self.n, 0), dtype=self.dtype, order="F")
        return self._get(3, (self.n, self.cols))

    @property
    def markers(self):
        out = np.zeros(max(1, self.cols), dtype=np.uint8)
        _check(load_library().rd_basis_markers(self.h, _p(out)))
        return out[: self.cols]

    def space(self, j) -> List[int]:
        m = load_library().rd_basis_space(self.h, j, None)
        out = np.zeros(max(m, 1), dtype=np.int32)
        load_library().rd_basis_space(self.h, j, _p(out))
        return out[:m].tolist()

    def get_into(self, which: int, out: np.ndarray) -> np.ndarray:
        """rd_basis_get into a caller-owned Fortran buffer with >= cols columns
        (0 V, 1 K_img, 3 W: n x cols; 2 R: cols x cols); returns the filled view."""
        r = self.cols
        shape = (r, r) if which == 2 else (self.n, r)
        if out.dtype != self.dtype or not out.flags.f_contiguous or out.shape[0] != shape[0] or out.shape[1] < r:
            raise ValueError("get_into: buffer must be Fortran-ordered, dtype %s, %d rows, >= %d cols"
                             % (self.dtype, shape[0], r))
        view = out[:, :r]
        _check(load_library().rd_basis_get(self.h, which, _p(view)))
        return view

    def set_rhs_hook(self, fn=None):
        """Checkpoint hook: fn(system_index, j) runs before RHS j of every
        process_system (the state it reads is the one the reference's loop body
        starts from). An exception in fn aborts the system (SolverError) and is
        re-raised from process_system's caller via ``hook_error``."""
        self.hook_error = None
        if fn is None:
            self._hook = None
            _check(load_library().rd_basis_set_rhs_hook(self.h, C.cast(None, RHS_HOOK), None))
            return

        def tramp(_user, system_index, j):
            try:
                fn(int(system_index), int(j))
                return 0
            except BaseException as e:  # noqa: BLE001 -- surfaced after the C call returns
                self.hook_error = e
                return 1

        self._hook = RHS_HOOK(tramp)
        _check(load_library().rd_basis_set_rhs_hook(self.h, self._hook, None))

    def compress(self, tol: float = 1e-10, normalize: bool = True):
        """Algorithm 1 compression in place (RRQR); V becomes the orthonormal
        retained basis. Returns (rank, perm, rdiag)."""
        m = self.cols
        rank = C.c_long()
        perm = np.zeros(max(m, 1), dtype=np.int64)
        rdiag = np.zeros(max(m, 1))
        _check(load_library().rd_basis_compress(self.h, tol, int(normalize), C.byref(rank), _p(perm), _p(rdiag)))
        return rank.value, perm[:m], rdiag[:m]

    def save(self, path: str):
        """write_basis of V and its markers (io.cpp:77-91; harness.cpp:194)."""
        _check(load_library().rd_basis_save(self.h, str(path).encode()))

    def refresh(self, op: SchurOperator):
        _check(load_library().rd_basis_refresh(self.h, op.h))

    def append(self, y, z, marker: int = 2) -> bool:
        y = np.ascontiguousarray(y, dtype=self.dtype)
        z = np.ascontiguousarray(z, dtype=self.dtype)
        ok = C.c_int()
        _check(load_library().rd_basis_append(self.h, _p(y), _p(z), marker, HOST, C.byref(ok)))
        return bool(ok.value)

    def solve_projected(self, b):
        b = np.ascontiguousarray(b, dtype=self.dtype)
        x = np.zeros(self.n, dtype=self.dtype)
        _check(load_library().rd_basis_solve_projected(self.h, _p(b), _p(x), None, HOST))
        return x

    def projected_coordinates(self, b):
        b = np.ascontiguousarray(b, dtype=self.dtype)
        x = np.zeros(self.n, dtype=self.dtype)
        c = np.zeros(self.cols, dtype=self.dtype)
        _check(load_library().rd_basis_solve_projected(self.h, _p(b), _p(x), _p(c), HOST))
        return c


def process_system(gb: GlobalBasis, op: SchurOperator, layout: P.Layout, tol: float, system_index: int,
                   maxit: int = 0, want_X: bool = True, X_out=None) -> ProcessResult:
    """Algorithm 2 main loop for one system (basis.cpp:157-207).

    X: a new host array when ``want_X``; ``X_out`` = a caller-owned host
    Fortran (n x nrhs) array (e.g. pinned memory) filled in place, or an int
    device pointer (n x nrhs, column-major) written on the device."""
    nrhs = layout.n_rhs
    idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
    val = np.ascontiguousarray(layout.val, dtype=np.float64)
    where = HOST
    if X_out is None:
        X = np.zeros((gb.n, nrhs), dtype=gb.dtype, order="F") if want_X else None
        xp = _p(X)
    elif isinstance(X_out, int):
        X, xp, where = None, C.c_void_p(X_out), DEVICE
    else:
        if X_out.dtype != gb.dtype or X_out.shape != (gb.n, nrhs) or not X_out.flags.f_contiguous:
            raise ValueError("process_system: X_out must be a Fortran (n, nrhs) array of the basis dtype")
        X, xp = X_out, _p(X_out)
    log = np.zeros((nrhs, 5))
    its, app = C.c_long(), C.c_long()
    rc = load_library().rd_process_system(gb.h, op.h, nrhs, _p(idx), _p(val), tol, system_index, maxit, xp,
                                          where, _p(log), C.byref(its), C.byref(app))
    if rc != 0 and getattr(gb, "hook_error", None) is not None:
        err, gb.hook_error = gb.hook_error, None
        raise err
    _check(rc)
    rows = [BuildLogRow(int(r[0]), int(r[1]), float(r[2]), int(r[3]), bool(r[4])) for r in log]
    return ProcessResult(X, rows, its.value, app.value)


class PerRhsRecycler(GlobalBasis):
    """BaselinePerRhsRecycler (basis.hpp:102-119, basis.cpp:209-266) on the
    device: per-RHS-only recycling, the paper's Table 2 comparator."""

    def __init__(self, U0: np.ndarray, X0: np.ndarray, ctx: Optional[Context] = None, dtype=None):
        self.ctx = ctx or default_context()
        dt = np.dtype(dtype) if dtype is not None else np.result_type(U0.dtype, X0.dtype)
        U0 = _f(U0, dt)
        X0 = _f(X0, dt)
        self.dtype = dt
        self.n = X0.shape[0]
        self.nrhs = X0.shape[1]
        h = C.c_void_p()
        _check(load_library().rd_per_rhs_create(self.ctx.h, _dt(dt), self.n, U0.shape[1], X0.shape[1], _p(U0),
                                                _p(X0), HOST, C.byref(h)))
        self.h = h

    def solve_system(self, op: SchurOperator, layout: P.Layout, tol: float, system_index: int, maxit: int = 0,
                     want_X: bool = True) -> ProcessResult:
        nrhs = layout.n_rhs
        idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
        val = np.ascontiguousarray(layout.val, dtype=np.float64)
        X = np.zeros((self.n, nrhs), dtype=self.dtype, order="F") if want_X else None
        log = np.zeros((nrhs, 5))
        its, app = C.c_long(), C.c_long()
        _check(load_library().rd_per_rhs_solve_system(self.h, op.h, nrhs, _p(idx), _p(val), tol, system_index, maxit,
                                                      _p(X), HOST, _p(log), C.byref(its), C.byref(app)))
        rows = [BuildLogRow(int(r[0]), int(r[1]), float(r[2]), int(r[3]), bool(r[4])) for r in log]
        return ProcessResult(X, rows, its.value, app.value)


def init_basis_from(U0, X0, cap: int = 0, ctx: Optional[Context] = None, dtype=None) -> GlobalBasis:
    """basis.cpp:114-134."""
    return GlobalBasis(U0, X0, cap, ctx, dtype)


def init_basis(op0: SchurOperator, op0_real: SchurOperator, layout: P.Layout, k_eig: int, tol: float,
               cap: int = 0, U0: Optional[np.ndarray] = None):
    """basis.cpp:136-155: U0 = k_eig smallest eigenvectors of the omega = 0
    operator (device Lanczos), X0 by CG/COCG at 0.25 tol."""
    lam = None
    if U0 is None:
        lam, U0 = smallest_eigenpairs(op0_real, k_eig, min(tol, 1e-8))
    X0, its = initial_solutions(op0, layout, tol)
    gb = GlobalBasis(U0.astype(op0.dtype), X0, cap, op0.ctx)
    return gb, X0, lam, U0


def bench_projection(n: int, c: int, cplx: bool, iters: int = 10, ctx: Optional[Context] = None):
    """Mean ms per launch of the three TMA projection kernels (C5 sweep hook)."""
    ctx = ctx or default_context()
    out = np.zeros(3)
    _check(load_library().rd_bench_projection(ctx.h, int(cplx), n, c, iters, _p(out)))
    return out


def bench_stencil(op: SchurOperator, ncols: int, iters: int = 10) -> float:
    out = np.zeros(1)
    _check(load_library().rd_bench_stencil(op.h, _dt(op.dtype), ncols, iters, _p(out)))
    return float(out[0])


def residual_norms(op: SchurOperator, layout: P.Layout, X, where: int = HOST) -> np.ndarray:
    """||b_j - A x_j|| / ||b_j|| per column, on the device (X host array or device pointer)."""
    idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
    val = np.ascontiguousarray(layout.val, dtype=np.float64)
    out = np.zeros(layout.n_rhs)
    xp = _p(_f(X, op.dtype)) if where == HOST else C.c_void_p(X)
    _check(load_library().rd_residual_norms(op.h, _dt(op.dtype), layout.n_rhs, _p(idx), _p(val), xp, where, _p(out)))
    return out


def rrqr(A: np.ndarray, tol: float = 1e-10, normalize: bool = True, ctx: Optional[Context] = None):
    ctx = ctx or default_context()
    A = _f(A, A.dtype)
    n, m = A.shape
    rank = C.c_long()
    perm = np.zeros(m, dtype=np.int64)
    rdiag = np.zeros(m)
    Q = np.zeros((n, m), dtype=A.dtype, order="F")
    _check(load_library().rd_rrqr(ctx.h, _dt(A.dtype), n, m, _p(A), tol, int(normalize), C.byref(rank), _p(perm),
                                  _p(rdiag), _p(Q), HOST))
    return rank.value, perm, rdiag, Q[:, : rank.value].copy()


def _csr(supports):
    ptr = np.zeros(len(supports) + 1, dtype=np.int64)
    for k, (ix, _) in enumerate(supports):
        ptr[k + 1] = ptr[k] + len(ix)
    if supports:
        sidx = np.ascontiguousarray(np.concatenate([np.asarray(ix, dtype=np.int64) for ix, _ in supports]))
        sval = np.ascontiguousarray(np.concatenate([np.asarray(w, dtype=np.float64) for _, w in supports]))
    else:
        sidx, sval = np.zeros(1, dtype=np.int64), np.zeros(1)
    if sidx.size == 0:
        sidx, sval = np.zeros(1, dtype=np.int64), np.zeros(1)
    return ptr, sidx, sval


def _layout_split(layout: P.Layout):
    idx = np.ascontiguousarray(layout.idx, dtype=np.int64)
    val = np.ascontiguousarray(layout.val, dtype=np.float64)
    s = layout.n_src
    return (np.ascontiguousarray(idx[:s]), np.ascontiguousarray(val[:s]),
            np.ascontiguousarray(idx[s:]), np.ascontiguousarray(val[s:]))


def fom_transfer(op: SchurOperator, layout: P.Layout, tol: float = 1e-10):
    """Full-order transfer C~^T A^-1 B~ (rom.cpp:86-91) by batched CG / COCG.
    Returns (Psi n_det x n_src, total iterations)."""
    si, sv, di, dv = _layout_split(layout)
    out = np.zeros((layout.n_det, layout.n_src), dtype=op.dtype, order="F")
    its = C.c_long()
    _check(load_library().rd_fom_transfer(op.h, _dt(op.dtype), layout.n_src, _p(si), _p(sv), layout.n_det, _p(di),
                                          _p(dv), tol, _p(out), HOST, C.byref(its)))
    return out, its.value


def fom_jacobian(op: SchurOperator, layout: P.Layout, supports, scale: float, tol: float = 1e-10):
    """Full-order Jacobian (rom.cpp:101-129): column k = scale * vec(sum_t w_t
    Z[i_t,:]^T X[i_t,:]) with X = A^-1 B~, Z = A^-1 C~; supports as in
    ReducedModel.jacobian."""
    si, sv, di, dv = _layout_split(layout)
    ptr, sidx, sval = _csr(supports)
    out = np.zeros((layout.n_det * layout.n_src, max(1, len(supports))), dtype=op.dtype, order="F")
    _check(load_library().rd_fom_jacobian(op.h, _dt(op.dtype), layout.n_src, _p(si), _p(sv), layout.n_det, _p(di),
                                          _p(dv), len(supports), _p(ptr), _p(sidx), _p(sval), float(scale), tol,
                                          _p(out), HOST))
    return out[:, : len(supports)]


class ReducedModel:
    """ReducedModel (include/romdot/rom.hpp:12-41, src/rom.cpp:9-67) on the device.

    V: host array (copied) or, with where=DEVICE, a device pointer that is
    borrowed and must outlive the model (e.g. a compressed GlobalBasis's V).
    Complex bases use bilinear projections (V^T A V, V^T B, V^T C)."""

    def __init__(self, V, dtype=None, ctx: Optional[Context] = None, where: int = HOST, n: int = 0, r: int = 0):
        self.ctx = ctx or default_context()
        if where == HOST:
            V = np.asfortranarray(V, dtype=dtype or np.asarray(V).dtype)
            self.dtype = V.dtype
            n, r = V.shape
            vp = _p(V)
        else:
            self.dtype = np.dtype(dtype)
            vp = C.c_void_p(V)
        self.n, self.r = int(n), int(r)
        h = C.c_void_p()
        _check(load_library().rd_rom_create(self.ctx.h, _dt(self.dtype), self.n, self.r, vp, where, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _release("rd_rom_destroy", self.h)
            except Exception:
                pass
            self.h = None

    def order(self) -> int:
        return load_library().rd_rom_order(self.h)

    @property
    def E_r(self) -> np.ndarray:
        out = np.zeros((self.r, self.r), dtype=self.dtype, order="F")
        _check(load_library().rd_rom_E(self.h, _p(out), HOST))
        return out

    def reduced_system(self, op: SchurOperator) -> np.ndarray:
        out = np.zeros((self.r, self.r), dtype=self.dtype, order="F")
        _check(load_library().rd_rom_reduced_system(self.h, op.h, _p(out), HOST))
        return out

    @staticmethod
    def _split(layout: P.Layout):
        return _layout_split(layout)

    def transfer(self, op: SchurOperator, layout: P.Layout) -> np.ndarray:
        """Psi_r = C_r^T A_r^-1 B_r, n_det x n_src."""
        si, sv, di, dv = self._split(layout)
        out = np.zeros((layout.n_det, layout.n_src), dtype=self.dtype, order="F")
        _check(load_library().rd_rom_transfer(self.h, op.h, layout.n_src, _p(si), _p(sv), layout.n_det, _p(di),
                                              _p(dv), _p(out), HOST))
        return out

    def jacobian(self, op: SchurOperator, layout: P.Layout, supports, scale: float) -> np.ndarray:
        """supports: one (index array, value array) pair per parameter (the
        reference's SparseDiag from absorption_jacobian); column k of the result
        is scale * vec(sum_t w_t (V Z)[i_t,:]^T (V Y)[i_t,:]), (n_det*n_src) x n_par."""
        si, sv, di, dv = self._split(layout)
        ptr, sidx, sval = _csr(supports)
        out = np.zeros((layout.n_det * layout.n_src, max(1, len(supports))), dtype=self.dtype, order="F")
        _check(load_library().rd_rom_jacobian(self.h, op.h, layout.n_src, _p(si), _p(sv), layout.n_det, _p(di),
                                              _p(dv), len(supports), _p(ptr), _p(sidx), _p(sval), float(scale),
                                              _p(out), HOST))
        return out[:, : len(supports)]


# ------------------------------------------------------------------ ROMB I/O --

def romb_write(path, V: np.ndarray, markers) -> None:
    """write_basis (io.cpp:77-91): version 1 for float64 (the reference's
    layout, bit-exact), version 2 with a dtype byte for complex128."""
    V = np.asfortranarray(V)
    if V.dtype not in (np.float64, np.complex128):
        raise ConfigError(2, "romb: float64 or complex128 only")
    mk = np.ascontiguousarray(np.asarray(markers, dtype=np.uint8))
    if mk.size != V.shape[1]:
        raise IoError(4, "basis file: marker count must equal column count")
    _check(load_library().rd_romb_write(str(path).encode(), _dt(V.dtype), V.shape[0], V.shape[1], _p(V),
                                        _p(mk) if mk.size else None, HOST, None))


def romb_info(path):
    dt, n, r = C.c_int(), C.c_long(), C.c_long()
    _check(load_library().rd_romb_info(str(path).encode(), C.byref(dt), C.byref(n), C.byref(r)))
    return (np.complex128 if dt.value == 1 else np.float64), n.value, r.value


def romb_read(path):
    """read_basis (io.cpp:93-110) -> (V, markers)."""
    dt, n, r = romb_info(path)
    V = np.zeros((n, r), dtype=dt, order="F")
    mk = np.zeros(max(r, 1), dtype=np.uint8)
    _check(load_library().rd_romb_read(str(path).encode(), _dt(dt), n, r, _p(V), _p(mk), HOST, None))
    return V, mk[:r].copy()


def bench_gram(n: int, a: int, b: int, cplx: bool, sym: bool, iters: int = 5, ctx: Optional[Context] = None) -> float:
    """Mean device ms of the tall Gram on seeded data (bench hook)."""
    ctx = ctx or default_context()
    ms = np.zeros(1)
    _check(load_library().rd_bench_gram(ctx.h, 1 if cplx else 0, n, a, b, int(sym), iters, _p(ms)))
    return float(ms[0])


def bench_gemm(n: int, a: int, b: int, cplx: bool, upper: bool = False, iters: int = 5,
               ctx: Optional[Context] = None) -> float:
    """Mean device ms of the tall GEMM X (n x a) M (a x b) on seeded data (bench hook)."""
    ctx = ctx or default_context()
    ms = np.zeros(1)
    _check(load_library().rd_bench_gemm(ctx.h, 1 if cplx else 0, n, a, b, int(upper), iters, _p(ms)))
    return float(ms[0])
