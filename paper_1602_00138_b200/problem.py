"""Host-side synthetic inputs for the basis build (generated once, the same
bytes feed the CUDA path and the CPU oracle).

* ``XorShift64Star`` / ``NormalStream`` -- bit-exact port of the reference's
  seeded generator (``proj/src/config.cpp:249-271``).
* ``evenly_spaced_positions`` -- ``proj/src/grid.cpp:107-121``.
* ``GridSpec`` -- the Schur-complement grid of ``proj/src/grid.cpp:38-160``,
  generalised to d = 2, 3: N_0 .. N_{d-2} lateral
  nodes with homogeneous Dirichlet ghosts, N_{d-1} interior layers along the
  Robin axis whose two boundary layers are eliminated.
* ``level_set_fields`` -- Gaussian-RBF level set, arctan Heaviside of
  ``proj/src/pals.cpp:11-13`` (App. A7), D = 1/(3(mu_a + mu_s')).
* ``CONFIGS`` -- BASELINE.json configs C1..C4 plus small
  parity configs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

_M64 = (1 << 64) - 1


class XorShift64Star:
    """xorshift64* with the top 53 bits mapped to (0, 1] (config.cpp:256-263)."""

    def __init__(self, seed: int):
        self.state = (seed & _M64) or 0x9E3779B97F4A7C15

    def uniform(self) -> float:
        s = self.state
        s ^= s >> 12
        s ^= (s << 25) & _M64
        s ^= s >> 27
        self.state = s
        z = (s * 0x2545F4914F6CDD1D) & _M64
        return ((z >> 11) + 1.0) * 2.0 ** -53


class NormalStream:
    """Box-Muller over XorShift64Star, spare kept (config.cpp:249-271)."""

    def __init__(self, seed: int):
        self.gen = XorShift64Star(seed)
        self.have_spare = False
        self.spare = 0.0

    def next(self) -> float:
        if self.have_spare:
            self.have_spare = False
            return self.spare
        u1 = self.gen.uniform()
        u2 = self.gen.uniform()
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = 2.0 * math.pi * u2
        self.spare = radius * math.sin(angle)
        self.have_spare = True
        return radius * math.cos(angle)


def _lround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def evenly_spaced_positions(nx: int, count: int) -> List[int]:
    """Evenly spaced indices excluding the corner nodes (grid.cpp:107-121)."""
    if count < 1 or count > nx - 2:
        raise ValueError("layout: source/detector count must be in [1, nx-2]")
    if count == 1:
        pos = [nx // 2]
    else:
        pos = [1 + _lround(k * (nx - 3) / (count - 1)) for k in range(count)]
    if len(set(pos)) != count:
        raise ValueError("layout: positions collide; too many sources/detectors for this grid")
    return pos


@dataclass
class GridSpec:
    """Interior-node grid of the eliminated-Robin Schur operator.

    ``N[-1]`` is the Robin axis. Node index p = i0 + N0*(i1 + N1*i2).
    Row scaling follows the reference (h^2-scaled rows, grid.cpp:66-75).
    """

    d: int
    N: Tuple[int, ...]
    h: float
    A: float = 1.0          # Robin reflection constant (GridConfig::boundary_constant)
    D_bg: float = 0.3       # diffusion of the boundary layer (reference: the constant D0)

    @property
    def n(self) -> int:
        return int(np.prod(self.N))

    @property
    def rho(self) -> float:
        return 2.0 * self.A * self.D_bg / self.h          # grid.cpp:44

    @property
    def robin_face(self) -> float:
        """Robin-face coefficient Dbg - Dbg*rho/(1+rho) = Dbg/(1+rho)."""
        return self.D_bg / (1.0 + self.rho)

    @property
    def b_src(self) -> float:
        # B~ = D2 (G^-1 B1) (grid.cpp:153-154), in the reference's operation order
        # (cwiseInverse of g_diag first), so the values equal the reference's bit for bit
        return -self.D_bg * (1.0 / (1.0 + self.rho))

    @property
    def c_det(self) -> float:
        return -self.rho * (1.0 / (1.0 + self.rho))       # C~ = D1^T (G^-1 C1) (grid.cpp:155)

    def node(self, *idx: int) -> int:
        p, stride = 0, 1
        for a, i in enumerate(idx):
            p += i * stride
            stride *= self.N[a]
        return p

    def coordinates(self) -> np.ndarray:
        """(n, d) node coordinates: lateral i*h, Robin-axis layer k*h."""
        axes = [np.arange(Na) * self.h for Na in self.N]
        mesh = np.meshgrid(*axes, indexing="ij")
        # flatten with axis 0 fastest
        return np.stack([m.transpose(*reversed(range(self.d))).reshape(-1) for m in mesh], axis=1)

    @staticmethod
    def reference_2d(nx: int, ny: int, b1: float = 4.0, diffusion: float = 0.3, A: float = 1.0) -> "GridSpec":
        """The reference's own 2D grid (grid.hpp:12-26): nx x (ny-2) unknowns, square cells."""
        if nx < 5 or ny < 5:
            raise ValueError("grid: nx and ny must both be at least 5")
        return GridSpec(d=2, N=(nx, ny - 2), h=b1 / (nx - 1), A=A, D_bg=diffusion)


@dataclass
class Layout:
    """Effective sources/detectors: one nonzero per column (grid.cpp:123-160)."""

    idx: np.ndarray   # int64 (n_rhs,) node index of each column, sources then detectors
    val: np.ndarray   # float64 (n_rhs,)
    n_src: int
    n_det: int

    @property
    def n_rhs(self) -> int:
        return int(self.idx.shape[0])

    def dense(self, n: int, dtype=np.float64) -> np.ndarray:
        B = np.zeros((n, self.n_rhs), dtype=dtype, order="F")
        B[self.idx, np.arange(self.n_rhs)] = self.val
        return B


def make_layout(grid: GridSpec, src: Sequence[int], det: Sequence[int], src_high: bool) -> Layout:
    """``src``/``det``: lattice counts per lateral axis (2D: (count,), 3D: (c0, c1)).

    2D reference convention: sources on the top row (Robin layer N-1 side),
    detectors on the bottom row. 3D (BASELINE): sources on z=0, detectors z=1.
    """
    last = grid.N[-1] - 1
    src_layer = last if src_high else 0
    det_layer = 0 if src_high else last

    def lattice(counts, layer):
        pos = [evenly_spaced_positions(grid.N[a], c) for a, c in enumerate(counts)]
        nodes = []
        if grid.d == 2:
            for i in pos[0]:
                nodes.append(grid.node(i, layer))
        else:
            for j in pos[1]:
                for i in pos[0]:
                    nodes.append(grid.node(i, j, layer))
        return nodes

    s = lattice(src, src_layer)
    t = lattice(det, det_layer)
    if len(set(s) | set(t)) != len(s) + len(t):
        raise ValueError("layout: source/detector nodes must be disjoint")
    idx = np.array(s + t, dtype=np.int64)
    val = np.array([grid.b_src] * len(s) + [grid.c_det] * len(t), dtype=np.float64)
    return Layout(idx=idx, val=val, n_src=len(s), n_det=len(t))


def smooth_heaviside(t, eps: float = 0.05):
    return 0.5 * (1.0 + (2.0 / math.pi) * np.arctan(t / eps))   # pals.cpp:11-13


@dataclass
class RBFParams:
    centres: np.ndarray   # (m, d)
    widths: np.ndarray    # (m,)


def draw_rbf(seed: int, m: int, d: int) -> RBFParams:
    g = XorShift64Star(seed)
    centres = np.array([[0.2 + 0.6 * g.uniform() for _ in range(d)] for _ in range(m)])
    widths = np.array([0.05 + 0.10 * g.uniform() for _ in range(m)])
    return RBFParams(centres, widths)


def perturb_rbf(p: RBFParams, seed: int, sigma: float = 0.05) -> RBFParams:
    """Interpolation point: centres and widths + N(0, sigma), widths >= 0.01 (App. A12)."""
    s = NormalStream(seed)
    c = p.centres.copy()
    w = p.widths.copy()
    for j in range(c.shape[0]):
        for a in range(c.shape[1]):
            c[j, a] += sigma * s.next()
        w[j] = max(0.01, w[j] + sigma * s.next())
    return RBFParams(c, w)


def perturb_rbf_reference(p: RBFParams, seed: int, jitter: float) -> RBFParams:
    """The reference's parameter sequence (harness.cpp:62-75): widths x (1 +
    0.01 N(0,1)), centres + jitter N(0,1) with jitter = 0.02 h (nx / 8); the
    amplitude draw (x (1 + 0.03 N)) is consumed to keep the stream aligned but
    this level-set model has unit amplitudes."""
    s = NormalStream(seed)
    c = p.centres.copy()
    w = p.widths.copy()
    for j in range(c.shape[0]):
        s.next()  # amplitude factor (p[j] *= 1 + 0.03 z)
        w[j] = w[j] * (1.0 + 0.01 * s.next())
        for a in range(c.shape[1]):
            c[j, a] += jitter * s.next()
    return RBFParams(c, w)


def absorption(grid: GridSpec, p: RBFParams, mu_bg: float = 0.01, contrast: float = 0.02,
               eps: float = 0.05) -> np.ndarray:
    """mu_a = mu_bg + contrast * H_eps(phi), phi = sum_j psi(|x-c_j|/w_j) - 1/2,
    psi(r) = exp(-r^2/2) 1[r < 3] (compactly supported Gaussian RBF)."""
    # separable squared distances broadcast over the (N_{d-1}, ..., N_0) node
    # array (C order = node order p = i0 + N0 (i1 + N1 i2)); summed axis 0
    # first, the same association as sum(axis=1) over (n, d) coordinates, so
    # the values are bit-identical to the coordinate-list form
    axes = [np.arange(Na) * grid.h for Na in grid.N]
    phi = np.full(grid.n, -0.5)
    for c, w in zip(p.centres, p.widths):
        r2 = None
        for a in range(grid.d):
            shape = [1] * grid.d
            shape[grid.d - 1 - a] = grid.N[a]
            da = ((axes[a] - c[a]) ** 2).reshape(shape)
            r2 = da if r2 is None else r2 + da
        r = np.sqrt(r2.reshape(-1)) / w
        phi += np.where(r < 3.0, np.exp(-0.5 * r * r), 0.0)
    return mu_bg + contrast * smooth_heaviside(phi, eps)


@dataclass
class Fields:
    """Per-system operator coefficients (device-ready float64 arrays)."""

    D: np.ndarray        # node diffusion
    mu: np.ndarray       # h^2 mu_a
    shift: float         # h^2 omega/nu (imaginary diagonal)


def fields_from_absorption(grid: GridSpec, mu_a: np.ndarray, omega_over_nu: float = 0.0,
                           mus_prime: float = 1.0) -> Fields:
    D = 1.0 / (3.0 * (mu_a + mus_prime))
    return Fields(D=np.ascontiguousarray(D, dtype=np.float64),
                  mu=np.ascontiguousarray(grid.h * grid.h * mu_a, dtype=np.float64),
                  shift=grid.h * grid.h * omega_over_nu)


def constant_fields(grid: GridSpec, mu_scaled: np.ndarray, D0: Optional[float] = None) -> Fields:
    """Reference mode: constant D0 everywhere, given h^2-scaled absorption."""
    D0 = grid.D_bg if D0 is None else D0
    return Fields(D=np.full(grid.n, D0), mu=np.ascontiguousarray(mu_scaled, dtype=np.float64), shift=0.0)


@dataclass
class ProblemConfig:
    name: str
    d: int
    N: int
    n_src: Tuple[int, ...]
    n_det: Tuple[int, ...]
    m_rbf: int
    n_points: int
    omegas: Tuple[float, ...]
    k: int
    tol: float = 1e-8
    complex: bool = False
    cap: int = 0
    seed: int = 20160200
    src_high: Optional[bool] = None
    mus_prime: float = 1.0
    ref_sequence: bool = False  # the reference's small per-system perturbations (harness.cpp:62-75)

    @property
    def grid(self) -> GridSpec:
        h = 1.0 / (self.N - 1)
        D_bg = 1.0 / (3.0 * (0.01 + self.mus_prime))
        return GridSpec(d=self.d, N=(self.N,) * self.d, h=h, A=1.0, D_bg=D_bg)

    @property
    def dtype(self):
        return np.complex128 if self.complex else np.float64

    def layout(self) -> Layout:
        high = (self.d == 2) if self.src_high is None else self.src_high
        return make_layout(self.grid, self.n_src, self.n_det, src_high=high)

    def base_params(self) -> RBFParams:
        return draw_rbf(self.seed, self.m_rbf, self.d)

    def point_params(self, i: int) -> RBFParams:
        """i = 0: unperturbed p0 (init_basis); i >= 1: perturbed interpolation points."""
        p0 = self.base_params()
        if i == 0:
            return p0
        if self.ref_sequence:
            jitter = 0.02 * self.grid.h * (self.N / 8.0)
            return perturb_rbf_reference(p0, self.seed + 1000003 * i, jitter)
        return perturb_rbf(p0, self.seed + 1000003 * i)   # harness.cpp:65 seed pattern

    def systems(self) -> List[Tuple[int, float]]:
        """Parameter-major (point, omega/nu) list of the K systems."""
        return [(i, w) for i in range(1, self.n_points + 1) for w in self.omegas]

    def fields(self, point: int, omega: float = 0.0) -> Fields:
        g = self.grid
        return fields_from_absorption(g, absorption(g, self.point_params(point)), omega, self.mus_prime)


CONFIGS = {
    # BASELINE.json configs
    "C1": ProblemConfig("C1", d=2, N=129, n_src=(16,), n_det=(16,), m_rbf=4, n_points=4, omegas=(0.0,), k=20),
    "C2": ProblemConfig("C2", d=2, N=513, n_src=(32,), n_det=(32,), m_rbf=6, n_points=6,
                        omegas=(0.0, 0.05, 0.1, 0.2), k=32, complex=True),
    "C3": ProblemConfig("C3", d=3, N=64, n_src=(4, 8), n_det=(4, 8), m_rbf=8, n_points=8, omegas=(0.0,), k=40),
    "C4": ProblemConfig("C4", d=3, N=128, n_src=(6, 8), n_det=(6, 8), m_rbf=12, n_points=8,
                        omegas=(0.0, 0.1), k=64, complex=True, cap=768),
    # the reference's acceptance criterion 5 (acceptance.cpp:314-334): 121^2 desk,
    # 32 + 32, 9 bumps, run defaults k_eig = 10, tol_basis = 1e-7 (config.hpp:42-46),
    # min(K, 2) systems (harness.cpp:224)
    "R5": ProblemConfig("R5", d=2, N=121, n_src=(32,), n_det=(32,), m_rbf=9, n_points=2, omegas=(0.0,), k=10,
                        tol=1e-7, ref_sequence=True),
    # R5 with another generator seed: over 12 seeds (20160200..20160211) the
    # checker's criterion-5 ratio spans 0.32 .. 0.69 (median 0.59); this one
    # gives 4098 / 9887 = 0.414, a case where the reference's own <= 0.5 bar
    # (acceptance.cpp:325) holds on the checker, so the device must meet it too
    "R5b": ProblemConfig("R5b", d=2, N=121, n_src=(32,), n_det=(32,), m_rbf=9, n_points=2, omegas=(0.0,), k=10,
                         tol=1e-7, ref_sequence=True, seed=20160209),
    # small parity configs (oracle finishes in seconds)
    "T2": ProblemConfig("T2", d=2, N=33, n_src=(4,), n_det=(4,), m_rbf=4, n_points=3, omegas=(0.0,), k=6),
    "T2c": ProblemConfig("T2c", d=2, N=33, n_src=(4,), n_det=(4,), m_rbf=4, n_points=2,
                         omegas=(0.0, 0.2), k=6, complex=True),
    "T3": ProblemConfig("T3", d=3, N=12, n_src=(2, 2), n_det=(2, 2), m_rbf=3, n_points=2, omegas=(0.0,), k=6),
    "T3c": ProblemConfig("T3c", d=3, N=12, n_src=(2, 2), n_det=(2, 2), m_rbf=3, n_points=2,
                         omegas=(0.0, 0.1), k=6, complex=True, cap=40),
}
