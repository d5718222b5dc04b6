"""ctypes wrapper of oracle/_ref/libromdot_ref.so -- THE REFERENCE ITSELF.
TEST INFRASTRUCTURE ONLY.

libromdot_ref.so is the reference's own library sources (proj/src/*.cpp)
compiled where they lie, unmodified, by ``make -C oracle _ref``; Eigen is
absent from this image, so they compile against oracle/eigen_shim (containers
and dense/sparse kernels written here, see its header) and are reached through
oracle/ref_driver.cpp (marshalling only).  Tests use it to pin the CPU
restatement (oracle.py / romdot_oracle.cpp) -- and through it the CUDA path --
to the reference's real control flow and arithmetic on the reference's own
problems (desk grids, PaLS absorption, harness parameter sequence).

Only tests/ and scripts/make_ref_golden.py import this module.  On a machine
without /root/reference the prebuilt .so (git-ignored, shipped by gpurun) is
used when present; ``available()`` says whether it can be loaded.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_ref", "libromdot_ref.so")
REFERENCE_ROOT = "/root/reference/proj"
_LIB = None


def build(force: bool = False) -> str:
    """Compile the reference from its sources (only where /root/reference exists)."""
    if os.path.isdir(REFERENCE_ROOT):
        deps = [os.path.join(_HERE, "ref_driver.cpp"), os.path.join(_HERE, "eigen_shim", "Eigen", "Core")]
        stale = not os.path.exists(_SO) or any(os.path.getmtime(d) > os.path.getmtime(_SO) for d in deps)
        if force or stale:
            subprocess.check_call(["make", "-s", "-C", _HERE, "_ref"])
    return _SO


def available() -> bool:
    try:
        build()
    except Exception:
        pass
    return os.path.exists(_SO)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ConfigError(RefError):
    pass


class SolverError(RefError):
    pass


class IoError(RefError):
    pass


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = C.CDLL(_SO)
        L.ref_last_error.restype = C.c_char_p
        for name in ("ref_grid_create", "ref_init_basis", "ref_init_basis_from", "ref_recycler_create",
                     "ref_rom_create", "ref_hybrid_create"):
            getattr(L, name).restype = C.c_void_p
        for name in ("ref_grid_dim", "ref_basis_cols", "ref_basis_ku", "ref_basis_full_solves", "ref_basis_space"):
            getattr(L, name).restype = C.c_long
        L.ref_grid_h.restype = C.c_double
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        raise {2: ConfigError, 3: SolverError, 4: IoError}.get(rc, RefError)(rc, msg)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f(a):
    return np.asfortranarray(a, dtype=np.float64)


def _v(a):
    return np.ascontiguousarray(a, dtype=np.float64)


vp, dbl, lng, cint = C.c_void_p, C.c_double, C.c_long, C.c_int


@dataclass
class Report:
    iterations: int
    converged: bool
    history: np.ndarray
    correction_norm: float = 0.0


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


def _rows(log):
    return [LogRow(int(r[0]), int(r[1]), float(r[2]), int(r[3]), bool(r[4])) for r in log]


def evenly_spaced_positions(nx: int, count: int) -> List[int]:
    pos = np.zeros(max(count, 1), dtype=np.int32)
    _check(lib().ref_evenly_spaced(cint(nx), cint(count), _p(pos)))
    return pos[:count].tolist()


class Grid:
    """Grid + assemble_blocks + SchurOperator (+ effective_layout) of grid.cpp."""

    def __init__(self, nx, ny, a1=0.0, b1=4.0, a3=0.0, b3=4.0, diffusion=0.3, boundary_constant=1.0):
        self.h_ = lib().ref_grid_create(cint(nx), cint(ny), dbl(a1), dbl(b1), dbl(a3), dbl(b3), dbl(diffusion),
                                        dbl(boundary_constant))
        if not self.h_:
            _check(2 if "grid" in lib().ref_last_error().decode() else 1)
        self.nx, self.ny = nx, ny
        self.n = lib().ref_grid_dim(vp(self.h_))
        self.h = lib().ref_grid_h(vp(self.h_))
        self.n_rhs = 0

    def __del__(self):
        if getattr(self, "h_", None):
            lib().ref_grid_free(vp(self.h_))
            self.h_ = None

    def interior_nodes(self):
        out = np.zeros((self.n, 2), order="F")
        _check(lib().ref_grid_interior_nodes(vp(self.h_), _p(out)))
        return out

    def apply(self, mu, x):
        mu, x = _v(mu), _v(x)
        y = np.zeros(self.n)
        _check(lib().ref_apply(vp(self.h_), _p(mu), _p(x), _p(y)))
        return y

    def matrix(self, mu):
        A = np.zeros((self.n, self.n), order="F")
        _check(lib().ref_with_absorption_dense(vp(self.h_), _p(_v(mu)), _p(A)))
        return A

    def full_block_matrix(self, mu):
        m = 2 * self.nx + self.n
        A = np.zeros((m, m), order="F")
        _check(lib().ref_full_block_matrix(vp(self.h_), _p(_v(mu)), _p(A)))
        return A

    def layout(self, src_positions, det_positions):
        s = np.ascontiguousarray(src_positions, dtype=np.int32)
        d = np.ascontiguousarray(det_positions, dtype=np.int32)
        B = np.zeros((self.n, s.size + d.size), order="F")
        _check(lib().ref_layout(vp(self.h_), cint(s.size), _p(s), cint(d.size), _p(d), _p(B)))
        self.n_src, self.n_det, self.n_rhs = int(s.size), int(d.size), int(s.size + d.size)
        return B

    def minres(self, mu, b, tol, maxit):
        mu, b = _v(mu), _v(b)
        x = np.zeros(self.n)
        its, conv, hl = cint(), cint(), lng()
        hist = np.zeros(maxit + 2)
        _check(lib().ref_minres(vp(self.h_), _p(mu), _p(b), dbl(tol), cint(maxit), _p(x), C.byref(its), C.byref(conv),
                                _p(hist), lng(hist.size), C.byref(hl)))
        return x, Report(its.value, bool(conv.value), hist[: hl.value].copy())

    def recycled_minres(self, mu, W, AW, rhs, tol, maxit, rhs_scale=0.0):
        mu, rhs, W, AW = _v(mu), _v(rhs), _f(W), _f(AW)
        corr, nd, im = np.zeros(self.n), np.zeros(self.n), np.zeros(self.n)
        its, conv, hl, cn = cint(), cint(), lng(), dbl()
        hist = np.zeros(maxit + 2)
        _check(lib().ref_recycled_minres(vp(self.h_), _p(mu), lng(W.shape[1]), _p(W), _p(AW), _p(rhs), dbl(tol),
                                         cint(maxit), dbl(rhs_scale), _p(corr), _p(nd), _p(im), C.byref(its),
                                         C.byref(conv), C.byref(cn), _p(hist), lng(hist.size), C.byref(hl)))
        return corr, nd, im, Report(its.value, bool(conv.value), hist[: hl.value].copy(), cn.value)

    def smallest_eigenpairs(self, mu, k, tol=1e-8):
        lam = np.zeros(k)
        U = np.zeros((self.n, k), order="F")
        _check(lib().ref_smallest_eigenpairs(vp(self.h_), _p(_v(mu)), cint(k), dbl(tol), _p(lam), _p(U)))
        return lam, U

    def fom_transfer(self, mu, minres=False, tol=1e-10):
        T = np.zeros((self.n_det, self.n_src), order="F")
        _check(lib().ref_fom_transfer(vp(self.h_), _p(_v(mu)), cint(int(minres)), dbl(tol), _p(T)))
        return T

    def fom_jacobian(self, pals: "Pals", p, nodes, h2, minres=False, tol=1e-10):
        J = np.zeros((self.n_src * self.n_det, 4 * pals.m_bumps), order="F")
        _check(lib().ref_fom_jacobian(vp(self.h_), cint(pals.m_bumps), _p(pals.prm), _p(_v(p)), _p(_f(nodes)), dbl(h2),
                                      cint(int(minres)), dbl(tol), _p(J)))
        return J


def minres_dense(A, b, tol, maxit):
    A, b = _f(A), _v(b)
    n = b.size
    x = np.zeros(n)
    its, conv, hl = cint(), cint(), lng()
    hist = np.zeros(maxit + 2)
    _check(lib().ref_minres_dense(lng(n), _p(A), _p(b), dbl(tol), cint(maxit), _p(x), C.byref(its), C.byref(conv),
                                  _p(hist), lng(hist.size), C.byref(hl)))
    return x, Report(its.value, bool(conv.value), hist[: hl.value].copy())


def from_raw(W, AW):
    W, AW = _f(W), _f(AW)
    U, K = np.zeros_like(W), np.zeros_like(W)
    _check(lib().ref_from_raw(lng(W.shape[0]), lng(W.shape[1]), _p(W), _p(AW), _p(U), _p(K)))
    return U, K


def from_raw_append(W, AW, u, k):
    W, AW = _f(W), _f(AW)
    n, c = W.shape
    U, K = np.zeros((n, c + 1), order="F"), np.zeros((n, c + 1), order="F")
    app = cint()
    _check(lib().ref_from_raw_append(lng(n), lng(c), _p(W), _p(AW), _p(_v(u)), _p(_v(k)), _p(U), _p(K), C.byref(app)))
    m = c + app.value
    return bool(app.value), U[:, :m], K[:, :m]


def initial_guess(W, AW, b):
    W, AW, b = _f(W), _f(AW), _v(b)
    z, r = np.zeros_like(b), np.zeros_like(b)
    _check(lib().ref_initial_guess(lng(W.shape[0]), lng(W.shape[1]), _p(W), _p(AW), _p(b), _p(z), _p(r)))
    return z, r


class Basis:
    """InitBasisResult: GlobalBasis + PerRhsSpaces (basis.hpp:28-79)."""

    def __init__(self, grid: Grid, handle):
        if not handle:
            msg = lib().ref_last_error().decode()
            raise SolverError(3, msg) if "failed" in msg or "converge" in msg else ConfigError(2, msg)
        self.g, self.h_ = grid, handle
        self.n = grid.n

    @classmethod
    def init(cls, grid: Grid, mu0, B, k_eig, tol):
        B = _f(B)
        return cls(grid, lib().ref_init_basis(vp(grid.h_), _p(_v(mu0)), _p(B), lng(B.shape[1]), cint(k_eig), dbl(tol)))

    @classmethod
    def init_from(cls, grid: Grid, U0, X0):
        U0, X0 = _f(U0), _f(X0)
        return cls(grid, lib().ref_init_basis_from(vp(grid.h_), _p(U0), lng(U0.shape[1]), _p(X0), lng(X0.shape[1])))

    def __del__(self):
        if getattr(self, "h_", None):
            lib().ref_basis_free(vp(self.h_))
            self.h_ = None

    @property
    def cols(self):
        return lib().ref_basis_cols(vp(self.h_))

    @property
    def eig_block(self):
        return lib().ref_basis_ku(vp(self.h_))

    @property
    def full_solves(self):
        return lib().ref_basis_full_solves(vp(self.h_))

    def _get(self, which, shape):
        out = np.zeros(shape, order="F")
        _check(lib().ref_basis_get(vp(self.h_), cint(which), _p(out)))
        return out

    V = property(lambda s: s._get(0, (s.n, s.cols)))
    K_img = property(lambda s: s._get(1, (s.n, s.cols)))
    R = property(lambda s: s._get(2, (s.cols, s.cols)))
    K_raw = property(lambda s: s._get(3, (s.n, s.cols)))
    Astar_V = property(lambda s: s._get(4, (s.n, s.cols)))

    def X0(self, nrhs):
        return self._get(5, (self.n, nrhs))

    @property
    def eigenvalues(self):
        return self._get(6, (self.eig_block,))

    @property
    def markers(self):
        out = np.zeros(self.cols, dtype=np.uint8)
        lib().ref_basis_markers(vp(self.h_), _p(out))
        return out

    def space(self, j):
        m = lib().ref_basis_space(vp(self.h_), lng(j), None)
        out = np.zeros(max(m, 1), dtype=np.int32)
        lib().ref_basis_space(vp(self.h_), lng(j), _p(out))
        return out[:m].tolist()

    def refresh(self, mu):
        _check(lib().ref_basis_refresh(vp(self.h_), _p(_v(mu))))

    def append(self, y, Astar_y, mu, marker=2):
        app = cint()
        _check(lib().ref_basis_append(vp(self.h_), _p(_v(y)), _p(_v(Astar_y)), _p(_v(mu)), cint(marker), C.byref(app)))
        return bool(app.value)

    def solve_projected(self, b):
        x, c = np.zeros(self.n), np.zeros(self.cols)
        _check(lib().ref_basis_solve_projected(vp(self.h_), _p(_v(b)), _p(x), _p(c)))
        return x

    def projected_coordinates(self, b):
        x, c = np.zeros(self.n), np.zeros(self.cols)
        _check(lib().ref_basis_solve_projected(vp(self.h_), _p(_v(b)), _p(x), _p(c)))
        return c

    def process_system(self, mu, B, tol, system_index, maxit=0):
        B = _f(B)
        nrhs = B.shape[1]
        X = np.zeros((self.n, nrhs), order="F")
        log = np.zeros((nrhs, 5))
        its, app = lng(), lng()
        _check(lib().ref_process_system(vp(self.h_), vp(self.g.h_), _p(_v(mu)), _p(B), lng(nrhs), dbl(tol),
                                        cint(system_index), cint(maxit), _p(X), _p(log), C.byref(its), C.byref(app)))
        return ProcessResult(X, _rows(log), its.value, app.value)


class PerRhsRecycler:
    """BaselinePerRhsRecycler (basis.cpp:209-266)."""

    def __init__(self, grid: Grid, U0, X0):
        U0, X0 = _f(U0), _f(X0)
        self.g, self.n = grid, grid.n
        self.h_ = lib().ref_recycler_create(vp(grid.h_), _p(U0), lng(U0.shape[1]), _p(X0), lng(X0.shape[1]))

    def __del__(self):
        if getattr(self, "h_", None):
            lib().ref_recycler_free(vp(self.h_))
            self.h_ = None

    def solve_system(self, mu, B, tol, system_index, maxit=0):
        B = _f(B)
        nrhs = B.shape[1]
        X = np.zeros((self.n, nrhs), order="F")
        log = np.zeros((nrhs, 5))
        its, app = lng(), lng()
        _check(lib().ref_recycler_solve_system(vp(self.h_), lng(self.n), _p(_v(mu)), _p(B), lng(nrhs), dbl(tol),
                                               cint(system_index), cint(maxit), _p(X), _p(log), C.byref(its),
                                               C.byref(app)))
        return ProcessResult(X, _rows(log), its.value, app.value)


def basis_coefficients(V, X):
    V, X = _f(V), _f(X)
    Cc = np.zeros((V.shape[1], X.shape[1]), order="F")
    _check(lib().ref_basis_coefficients(lng(V.shape[0]), lng(V.shape[1]), _p(V), lng(X.shape[1]), _p(X), _p(Cc)))
    return Cc


class Pals:
    """PalsModel (pals.hpp:11-27) with the reference's defaults."""

    def __init__(self, m_bumps=9, mu_in=0.5, mu_out=0.05, eps_heaviside=0.05, eps_norm=4e-3, level=0.0):
        self.m_bumps = m_bumps
        self.prm = np.array([mu_in, mu_out, eps_heaviside, eps_norm, level], dtype=np.float64)

    def absorption(self, p, nodes):
        nodes = _f(nodes)
        mu = np.zeros(nodes.shape[0])
        _check(lib().ref_pals_absorption(cint(self.m_bumps), _p(self.prm), _p(_v(p)), lng(nodes.shape[0]), _p(nodes),
                                         _p(mu)))
        return mu

    def jacobian_column(self, p, k, nodes):
        nodes = _f(nodes)
        col = np.zeros(nodes.shape[0])
        _check(lib().ref_pals_jacobian_column(cint(self.m_bumps), _p(self.prm), _p(_v(p)), cint(k),
                                              lng(nodes.shape[0]), _p(nodes), _p(col)))
        return col


class ReducedModel:
    """ReducedModel (rom.cpp:9-67) on grid.layout()'s B~ / C~."""

    def __init__(self, grid: Grid, V):
        V = _f(V)
        self.g, self.r = grid, V.shape[1]
        self.h_ = lib().ref_rom_create(vp(grid.h_), _p(V), lng(V.shape[1]))
        if not self.h_:
            msg = lib().ref_last_error().decode()
            raise SolverError(3, msg) if "rank" in msg else ConfigError(2, msg)

    def __del__(self):
        if getattr(self, "h_", None):
            lib().ref_rom_free(vp(self.h_))
            self.h_ = None

    def reduced_system(self, mu):
        A = np.zeros((self.r, self.r), order="F")
        _check(lib().ref_rom_reduced_system(vp(self.h_), lng(self.g.n), _p(_v(mu)), _p(A)))
        return A

    def transfer(self, mu):
        T = np.zeros((self.g.n_det, self.g.n_src), order="F")
        _check(lib().ref_rom_transfer(vp(self.h_), lng(self.g.n), _p(_v(mu)), _p(T)))
        return T

    def jacobian(self, pals: Pals, p, nodes, h2):
        J = np.zeros((self.g.n_src * self.g.n_det, 4 * pals.m_bumps), order="F")
        _check(lib().ref_rom_jacobian(vp(self.h_), cint(pals.m_bumps), _p(pals.prm), _p(_v(p)), lng(self.g.n),
                                      _p(_f(nodes)), dbl(h2), _p(J)))
        return J


# ---- experiment layer (config.cpp / harness.cpp / io.cpp / inversion.cpp) ----

def exp_config(nx=-1, ny=-1, n_src=-1, n_det=-1, m_bumps=-1, seed=-1, k_systems=-1, k_eig=-1, tol_basis=-1.0):
    """ExperimentConfig with the reference's defaults; -1 keeps a default."""
    return np.array([nx, ny, n_src, n_det, m_bumps, seed, k_systems, k_eig, tol_basis], dtype=np.float64)


def exp_dims(cfg):
    d = (lng * 3)()
    _check(lib().ref_exp_dims(_p(cfg), d))
    return int(d[0]), int(d[1]), int(d[2])


def exp_parameters(cfg, index):
    p = np.zeros(exp_dims(cfg)[2])
    _check(lib().ref_exp_parameters(_p(cfg), cint(index), _p(p)))
    return p


def exp_mu(cfg, index):
    """(h^2 mu of parameter_in_sequence(cfg, index), B_concat) as cmd_compare_recycling forms them."""
    n, nrhs, _ = exp_dims(cfg)
    mu = np.zeros(n)
    B = np.zeros((n, nrhs), order="F")
    _check(lib().ref_exp_mu(_p(cfg), cint(index), _p(mu), _p(B)))
    return mu, B


def compare_recycling(cfg, out_dir):
    """cmd_compare_recycling: (shared-basis, per-RHS-only) inner iteration totals."""
    ours, base = lng(), lng()
    _check(lib().ref_compare_recycling(_p(cfg), out_dir.encode(), C.byref(ours), C.byref(base)))
    return ours.value, base.value


def normal_stream(seed, count):
    out = np.zeros(count)
    _check(lib().ref_normal_stream(C.c_uint64(seed), lng(count), _p(out)))
    return out


def offline_hash(cfg):
    buf = C.create_string_buffer(256)
    _check(lib().ref_offline_hash(_p(cfg), buf, lng(256)))
    return buf.value.decode()


def format_sci(v):
    buf = C.create_string_buffer(64)
    _check(lib().ref_format_sci(dbl(v), buf, lng(64)))
    return buf.value.decode()


def write_basis(path, V, markers):
    V = _f(V)
    mk = np.ascontiguousarray(markers, dtype=np.uint8)
    _check(lib().ref_write_basis(path.encode(), lng(V.shape[0]), lng(V.shape[1]), _p(V), _p(mk)))


def read_basis(path):
    n, r = lng(), lng()
    _check(lib().ref_read_basis(path.encode(), C.byref(n), C.byref(r), None, None))
    V = np.zeros((n.value, r.value), order="F")
    mk = np.zeros(r.value, dtype=np.uint8)
    _check(lib().ref_read_basis(path.encode(), C.byref(n), C.byref(r), _p(V), _p(mk)))
    return V, mk


class HybridEvaluator:
    """HybridEvaluator (inversion.cpp:53-106) seeded by init_basis at parameter_in_sequence(cfg, 0)."""

    def __init__(self, cfg):
        self.cfg = cfg
        self.n, self.n_rhs, self.n_params = exp_dims(cfg)
        self.n_src, self.n_det = int(cfg[2]) if cfg[2] >= 0 else 8, int(cfg[3]) if cfg[3] >= 0 else 8
        self.h_ = lib().ref_hybrid_create(_p(cfg))
        if not self.h_:
            raise RefError(1, lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h_", None):
            lib().ref_hybrid_free(vp(self.h_))
            self.h_ = None

    def transfer(self, p):
        T = np.zeros((self.n_det, self.n_src), order="F")
        _check(lib().ref_hybrid_transfer(vp(self.h_), _p(_v(p)), _p(T)))
        return T

    def jacobian(self, p):
        J = np.zeros((self.n_src * self.n_det, self.n_params), order="F")
        _check(lib().ref_hybrid_jacobian(vp(self.h_), _p(_v(p)), _p(J)))
        return J

    def state(self):
        st = (lng * 6)()
        _check(lib().ref_hybrid_state(vp(self.h_), st))
        keys = ["cols", "systems_used", "appends", "in_rom_mode", "full_order_solves", "log_rows"]
        return dict(zip(keys, (int(x) for x in st)))

    def build_log(self):
        m = self.state()["log_rows"]
        log = np.zeros((max(m, 1), 5))
        _check(lib().ref_hybrid_log(vp(self.h_), _p(log)))
        return _rows(log[:m])

    def basis_V(self):
        V = np.zeros((self.n, self.state()["cols"]), order="F")
        _check(lib().ref_hybrid_basis_V(vp(self.h_), _p(V)))
        return V
