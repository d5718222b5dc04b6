"""Offline seed cache (cmd_offline, harness.cpp:254-293): the init_basis seed
(U0 = k smallest eigenvectors of the omega = 0 operator, X0 = the initial
solutions at 0.25 tol) computed on the device once per configuration and
cached as u0.romb / x0.romb with a key=value manifest keyed by an FNV-1a hash
of the configuration (config.cpp:205-218); a later build loads it and goes
straight to init_basis_from (basis.cpp:114-134).
"""
import os
from typing import Dict, Tuple

import numpy as np

from . import problem as P
from . import romdot as R

COL_EIGENVECTOR, COL_INITIAL_SOLUTION, COL_CORRECTION = 0, 1, 2   # basis.hpp:13-15


def format_sci(v: float) -> str:
    """io.cpp:11-15: printf("%.5e")."""
    return "%.5e" % v


def _num(v) -> str:
    return repr(float(v)) if isinstance(v, float) else str(v)


def config_hash(cfg: P.ProblemConfig) -> str:
    """FNV-1a over the fields that define the seed (the reference hashes its
    grid / layout / PaLS / k_eig / tolerance strings, config.cpp:205-218)."""
    h = 0xcbf29ce484222325
    fields = [cfg.d, cfg.N, tuple(cfg.n_src), tuple(cfg.n_det), cfg.m_rbf, cfg.k, cfg.seed, cfg.mus_prime,
              cfg.complex, cfg.src_high, cfg.grid.h, cfg.grid.D_bg]
    for t in fields:
        for byte in (_num(t) + "\x00").encode():
            h ^= byte
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def write_manifest(path: str, entries: Dict[str, str]) -> None:
    """io.cpp:112-117: key=value lines (sorted like std::map)."""
    try:
        with open(path, "w") as f:
            for k in sorted(entries):
                f.write(f"{k}={entries[k]}\n")
    except OSError as e:
        raise R.IoError(4, f"cannot open {path} for writing") from e


def read_manifest(path: str) -> Dict[str, str]:
    """io.cpp:119-131: '#' comments and blank lines skipped; a line without
    '=' is an IoError."""
    try:
        lines = open(path).read().splitlines()
    except OSError as e:
        raise R.IoError(4, f"cannot open {path}") from e
    out = {}
    for line in lines:
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise R.IoError(4, f"{path}: malformed manifest line: {line}")
        k, v = line.split("=", 1)
        out[k] = v
    return out


def offline_seed(cfg: P.ProblemConfig, out_dir: str, ctx=None) -> bool:
    """cmd_offline: True when valid cached artifacts exist (nothing computed),
    False after computing and writing them."""
    os.makedirs(out_dir, exist_ok=True)
    man = os.path.join(out_dir, "offline_manifest.txt")
    u0p, x0p = os.path.join(out_dir, "u0.romb"), os.path.join(out_dir, "x0.romb")
    h = config_hash(cfg)
    if os.path.exists(man) and os.path.exists(u0p) and os.path.exists(x0p):
        m = read_manifest(man)
        if m.get("hash") == h and m.get("tol_basis") == format_sci(cfg.tol):
            return True
    g, lay = cfg.grid, cfg.layout()
    f0 = cfg.fields(0)
    op0r = R.SchurOperator(g, f0, np.float64, ctx)
    op0 = R.SchurOperator(g, f0, cfg.dtype, ctx)
    _, U0 = R.smallest_eigenpairs(op0r, cfg.k, min(cfg.tol, 1e-8))
    X0, _ = R.initial_solutions(op0, lay, cfg.tol)
    R.romb_write(u0p, U0, [COL_EIGENVECTOR] * U0.shape[1])
    R.romb_write(x0p, X0, [COL_INITIAL_SOLUTION] * X0.shape[1])
    write_manifest(man, {"hash": h, "k_eig": str(cfg.k), "tol_basis": format_sci(cfg.tol), "n": str(g.n)})
    return False


def load_seed(out_dir: str) -> Tuple[np.ndarray, np.ndarray]:
    U0, mu = R.romb_read(os.path.join(out_dir, "u0.romb"))
    X0, mx = R.romb_read(os.path.join(out_dir, "x0.romb"))
    if np.any(mu != COL_EIGENVECTOR) or np.any(mx != COL_INITIAL_SOLUTION):
        raise R.IoError(4, f"{out_dir}: seed files carry unexpected column markers")
    return U0, X0
