"""Checkpoint-replay lockstep of the device basis build against the CPU
checker. TEST INFRASTRUCTURE ONLY (tests/, bench.py's reference / cpu_baseline
legs and scripts/ import it; the product package never does).

The reference's own record-then-replay pattern (proj/tests/acceptance.cpp:
201-250) applied at the target scale: the DEVICE runs the whole build
(process_system, proj/src/basis.cpp:157-207); before each sampled RHS j of a
sampled system, the rd_basis_set_rhs_hook checkpoint copies the basis state
the reference's loop body starts from (V, K_img, R, U_j's indices) to host
memory, and the checker replays that single RHS on the host cores
(orc.replay_rhs: global check, from_raw, recycled CG/COCG to 0.25 tol,
X_j = correction + solve_projected(b_j), append decision). After the system,
the device's BuildLog row j and solution X_j are compared with the replay:
identical append flags, iterations +-2, init_relres and X_j within 1e-6
(SURVEY App. C.2). The checker never holds K~ = A_i V (the reference's third
n x r matrix): A_i U_j is recomputed per RHS, so the C4 state at the
768-column cap (V + K_img = 51.6 GB complex128) fits the GPU box's host RAM.

Optional factor checks at a checkpoint use the checker's operator:
||K_img R - A_i V|| / ||A_i V|| on sampled columns and ||K_img^H K_img - I||
(full Gram, chunked) -- the refresh / append invariants of basis.cpp:37-103.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

import oracle as orc


@dataclass
class Checkpoint:
    system: int
    rhs: int
    cols: int
    space: List[int]
    replay: orc.ReplayResult
    copy_s: float
    device_row: Optional[tuple] = None      # (init_relres, iterations, appended)
    x_reldiff: Optional[float] = None
    x_residual_gpu: Optional[float] = None
    x_residual_cpu: Optional[float] = None


def default_points(n_systems: int, nrhs: int, n_src: int, per_system: int = 2) -> Dict[int, List[int]]:
    """Deterministic sample: per system one source and one detector RHS (and
    more if asked), spread over the index range."""
    pts = {}
    for s in range(1, n_systems + 1):
        js = [(7 * s + 3) % n_src, n_src + (11 * s + 5) % (nrhs - n_src)]
        k = 2
        while len(js) < per_system:
            js.append((js[-1] + 13 * k) % nrhs)
            k += 1
        pts[s] = sorted(set(js))[:per_system]
    return pts


def factor_checks(op_o: orc.Operator, V: np.ndarray, K: np.ndarray, R: np.ndarray, ncols: int = 16,
                  gram: bool = True, chunk: int = 1 << 16) -> dict:
    """Refresh-factor invariants with the checker's operator: K_img R = A_i V
    on ncols sampled columns (first, last, spread), K_img^H K_img = I."""
    n, r = V.shape
    cols = sorted(set(np.linspace(0, r - 1, ncols).astype(int).tolist()))
    AV = op_o.apply(np.asfortranarray(V[:, cols]))
    KR = K @ R[:, cols]
    fac = float(np.linalg.norm(KR - AV) / np.linalg.norm(AV))
    out = {"cols": r, "factor_cols_checked": len(cols), "KR_minus_AV_rel": fac}
    if gram:
        G = np.zeros((r, r), dtype=K.dtype)
        for i0 in range(0, n, chunk):
            B = np.ascontiguousarray(K[i0:i0 + chunk])
            G += B.conj().T @ B
        out["KhK_minus_I_max"] = float(np.abs(G - np.eye(r)).max())
    return out


class Sampler:
    """rd_basis_set_rhs_hook callback: replays the sampled (system, RHS) points
    on the checker and keeps the results for the post-system comparison."""

    def __init__(self, gb, cfg, layout, points: Dict[int, List[int]], cap: int, tol: float,
                 factor_check_systems: Sequence[int] = (), gram_check_systems: Sequence[int] = (),
                 keep_x: bool = True, verbose: bool = True):
        self.gb, self.cfg, self.lay = gb, cfg, layout
        self.points = {int(s): set(int(j) for j in js) for s, js in points.items()}
        self.cap, self.tol = cap, tol
        self.factor_systems = set(factor_check_systems)
        self.gram_systems = set(gram_check_systems)
        self.keep_x = keep_x
        self.verbose = verbose
        self.op_o: Optional[orc.Operator] = None
        self.results: List[Checkpoint] = []
        self.factor: Dict[int, dict] = {}
        ncap = max(cap, gb.cols) if cap else gb.cols + layout.n_rhs * max(1, len(cfg.systems()))
        self.ncap = ncap
        self.Vb = np.empty((gb.n, ncap), dtype=gb.dtype, order="F")
        self.Kb = np.empty((gb.n, ncap), dtype=gb.dtype, order="F")
        self.cpu_s = 0.0

    def set_operator(self, op_o: orc.Operator):
        self.op_o = op_o

    def __call__(self, system: int, j: int):
        if j not in self.points.get(system, ()):
            if j == 0 and system in self.factor_systems:
                self._factor(system)
            return
        t0 = time.perf_counter()
        r = self.gb.cols
        if r > self.ncap:
            raise RuntimeError("replay: basis wider than the host buffers")
        V = self.gb.get_into(0, self.Vb)
        K = self.gb.get_into(1, self.Kb)
        R = self.gb.R
        space = self.gb.space(j)
        t1 = time.perf_counter()
        if j == 0 and system in self.factor_systems:
            self._factor(system, V, K, R)
        res = orc.replay_rhs(self.op_o, V, K, R, space, int(self.lay.idx[j]), float(self.lay.val[j]), self.tol,
                             self.cap)
        self.cpu_s += res.times["total"]
        if not self.keep_x:
            res.X = None
        self.results.append(Checkpoint(system, j, r, space, res, t1 - t0))
        if self.verbose:
            import json
            import sys
            print(json.dumps({"replay": [system, j], "cols": r, "cj": len(space), "its": res.iterations,
                              "appended": res.appended, "init_relres": res.init_relres,
                              "cpu_s": round(res.times["total"], 2)}), file=sys.stderr, flush=True)

    def _factor(self, system, V=None, K=None, R=None):
        if V is None:
            V = self.gb.get_into(0, self.Vb)
            K = self.gb.get_into(1, self.Kb)
            R = self.gb.R
        t0 = time.perf_counter()
        fc = factor_checks(self.op_o, V, K, R, gram=system in self.gram_systems)
        fc["check_s"] = time.perf_counter() - t0
        self.factor[system] = fc

    def compare_system(self, system: int, log, X: Optional[np.ndarray]):
        """Attach the device row / X_j to this system's checkpoints."""
        for cp in self.results:
            if cp.system != system or cp.device_row is not None:
                continue
            row = log[cp.rhs]
            cp.device_row = (row.init_relres, row.iterations, row.appended)
            if X is not None and cp.replay.X is not None:
                xg = X[:, cp.rhs]
                xc = cp.replay.X
                cp.x_reldiff = float(np.linalg.norm(xg - xc) / np.linalg.norm(xc))
                b = np.zeros(self.gb.n, dtype=self.gb.dtype)
                b[self.lay.idx[cp.rhs]] = self.lay.val[cp.rhs]
                bn = np.linalg.norm(b)
                cp.x_residual_gpu = float(np.linalg.norm(self.op_o.apply(xg) - b) / bn)
                cp.x_residual_cpu = float(np.linalg.norm(self.op_o.apply(xc) - b) / bn)
                cp.replay.X = None  # keep memory bounded

    def summary(self) -> dict:
        done = [cp for cp in self.results if cp.device_row is not None]
        flips = [cp for cp in done if cp.device_row[2] != cp.replay.appended]
        its = [abs(cp.device_row[1] - cp.replay.iterations) for cp in done]
        rel = [abs(cp.device_row[0] - cp.replay.init_relres) / cp.replay.init_relres for cp in done
               if cp.replay.init_relres > 0]
        xd = [cp.x_reldiff for cp in done if cp.x_reldiff is not None]
        rg = [cp.x_residual_gpu for cp in done if cp.x_residual_gpu is not None]
        rc = [cp.x_residual_cpu for cp in done if cp.x_residual_cpu is not None]
        return {
            "rows": len(done),
            "systems": sorted({cp.system for cp in done}),
            "append_flips": len(flips),
            "max_iteration_diff": max(its) if its else None,
            "max_init_relres_reldiff": max(rel) if rel else None,
            "max_solution_reldiff": max(xd) if xd else None,
            "max_explicit_residual_gpu": max(rg) if rg else None,
            "max_explicit_residual_cpu": max(rc) if rc else None,
            "all_converged": all(cp.replay.converged for cp in done),
            "rows_detail": [[cp.system, cp.rhs, cp.cols, len(cp.space), cp.replay.iterations, cp.device_row[1],
                             int(cp.replay.appended), int(cp.device_row[2]), cp.replay.init_relres,
                             cp.device_row[0], cp.x_reldiff, round(cp.replay.times["total"], 3)] for cp in done],
            "rows_detail_cols": ["system", "rhs", "cols", "cj", "its_cpu", "its_gpu", "app_cpu", "app_gpu",
                                 "init_relres_cpu", "init_relres_gpu", "x_reldiff", "cpu_s"],
            "factor_checks": self.factor,
        }


def run_device_build(cfg, points: Dict[int, List[int]], systems: Optional[Sequence[int]] = None,
                     factor_check_systems: Sequence[int] = (), gram_check_systems: Sequence[int] = (),
                     seed_check: bool = True, verbose: bool = True, log=None) -> Tuple[dict, "Sampler"]:
    """Device seed + build of cfg's systems (1-based indices in ``systems``,
    default all) with checkpoint replay at ``points``. Returns (summary, sampler)."""
    import json
    import sys

    from paper_1602_00138_b200 import problem as P  # noqa: F401
    from paper_1602_00138_b200 import romdot as R

    def say(**kw):
        if verbose:
            print(json.dumps(kw), file=sys.stderr, flush=True)

    g, lay = cfg.grid, cfg.layout()
    t0 = time.perf_counter()
    f0 = cfg.fields(0)
    lam, U0 = R.smallest_eigenpairs(R.SchurOperator(g, f0, np.float64), cfg.k, min(cfg.tol, 1e-8))
    X0, _ = R.initial_solutions(R.SchurOperator(g, f0, cfg.dtype), lay, cfg.tol)
    out = {"seed_s": time.perf_counter() - t0}
    if seed_check:  # the device seed, checked with the checker's own operator
        op_r = orc.Operator.grid(g, f0)
        er = np.linalg.norm(op_r.apply(U0) - U0 * lam, axis=0)
        out["eig_residual_over_lammax"] = float(er.max() / op_r.lam_max)
        op0 = orc.Operator.grid(g, f0, cfg.dtype)
        res = []
        for j in range(lay.n_rhs):
            b = np.zeros(g.n, dtype=cfg.dtype)
            b[lay.idx[j]] = lay.val[j]
            res.append(np.linalg.norm(op0.apply(X0[:, j]) - b) / abs(lay.val[j]))
        out["X0_max_explicit_residual"] = float(max(res))
        del op_r, op0
    gb = R.GlobalBasis(U0.astype(cfg.dtype), X0, cfg.cap)
    del U0, X0
    smp = Sampler(gb, cfg, lay, points, cfg.cap, cfg.tol, factor_check_systems, gram_check_systems,
                  verbose=verbose)
    gb.set_rhs_hook(smp)
    all_sys = cfg.systems()
    todo = list(systems) if systems else list(range(1, len(all_sys) + 1))
    last = max(todo)
    sys_rows = []
    for s in range(1, last + 1):
        pt, w = all_sys[s - 1]
        f = cfg.fields(pt, w)
        smp.set_operator(orc.Operator.grid(g, f, cfg.dtype))
        if s not in todo:
            smp.points.pop(s, None)
        t1 = time.perf_counter()
        pr = R.process_system(gb, R.SchurOperator(g, f, cfg.dtype), lay, cfg.tol, s,
                              want_X=bool(smp.points.get(s)))
        smp.compare_system(s, pr.log, pr.X)
        sys_rows.append({"system": s, "omega": w, "cols": gb.cols, "its": pr.inner_iterations,
                         "appends": pr.appends, "wall_s": round(time.perf_counter() - t1, 2)})
        say(system=s, cols=gb.cols, its=pr.inner_iterations, appends=pr.appends)
        del pr
    gb.set_rhs_hook(None)
    out["systems"] = sys_rows
    out.update(smp.summary())
    out["cpu_replay_s"] = smp.cpu_s
    return out, smp
