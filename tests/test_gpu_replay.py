"""Checkpoint-replay lockstep of the device build against the CPU checker
(oracle/replay.py; the reference's record-then-replay pattern,
proj/tests/acceptance.cpp:201-250, at the BASELINE configs).

The device runs process_system (proj/src/basis.cpp:157-207) through the C ABI;
before a sampled RHS j, the rd_basis_set_rhs_hook checkpoint hands the basis
state (V, K_img, R, U_j) to the checker, which replays that RHS on the host
cores. Tolerances (north_star / SURVEY App. C.2), per replayed row:
  * identical append decision,
  * inner iterations within +-2,
  * init_relres within 1e-6 relative,
  * solution X_j within 1e-6 relative of the checker's,
  * explicit residual ||b_j - A X_j|| / ||b_j|| <= tol with the checker's operator.
"""
import numpy as np
import pytest

import oracle as orc
import replay as RP
from paper_1602_00138_b200 import problem as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    from paper_1602_00138_b200 import build, romdot
    build.build()
    return romdot


def check(out, tol, rows_min):
    assert out["rows"] >= rows_min, out
    assert out["all_converged"], out
    assert out["append_flips"] == 0, out
    assert out["max_iteration_diff"] <= 2, out
    assert out["max_init_relres_reldiff"] <= 1e-6, out
    assert out["max_solution_reldiff"] <= 1e-6, out
    assert out["max_explicit_residual_gpu"] <= tol, out
    assert out["max_explicit_residual_cpu"] <= tol, out


@pytest.mark.parametrize("name", ["T2c", "T3c"])
def test_replay_every_row(rd, name):
    """Every RHS of every system replayed (T3c reaches its 40-column cap)."""
    c = P.CONFIGS[name]
    lay = c.layout()
    pts = {s: list(range(lay.n_rhs)) for s in range(1, len(c.systems()) + 1)}
    out, _ = RP.run_device_build(c, pts, factor_check_systems=[1, len(c.systems())],
                                 gram_check_systems=[len(c.systems())], verbose=False)
    check(out, c.tol, len(c.systems()) * lay.n_rhs)
    assert out["eig_residual_over_lammax"] <= 1e-8
    assert out["X0_max_explicit_residual"] <= c.tol
    for fc in out["factor_checks"].values():
        assert fc["KR_minus_AV_rel"] <= 1e-12, fc
        assert fc.get("KhK_minus_I_max", 0.0) <= 1e-12, fc


def test_replay_c4_rows(rd):
    """Target config C4 (3D 128^3, complex128, k = 64, 96 RHS): one source RHS
    of system 1 (omega = 0) and one detector RHS of system 2 (omega/nu = 0.1,
    COCG) replayed on the host cores from the device's state, plus the refresh
    factor K_img R = A_2 V of system 2 with the checker's operator."""
    c = P.CONFIGS["C4"]
    lay = c.layout()
    pts = {1: [5], 2: [lay.n_src + 17]}
    out, _ = RP.run_device_build(c, pts, systems=[1, 2], factor_check_systems=[2], verbose=False)
    check(out, c.tol, 2)
    assert out["eig_residual_over_lammax"] <= 1e-8, out
    assert out["X0_max_explicit_residual"] <= c.tol, out
    assert out["factor_checks"][2]["KR_minus_AV_rel"] <= 1e-12, out["factor_checks"]


def test_c3_lockstep_two_full_systems(rd):
    """C3 (3D 64^3, real, 64 RHS): two whole systems in lockstep from the
    device seed -- every BuildLog row (append flags, +-2 iterations,
    init_relres), every solution's explicit residual, X within 1e-6."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "parity_full", os.path.join(os.path.dirname(__file__), "..", "scripts", "parity_full.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    out = mod.run("C3", n_systems=2, device_seed=True)
    assert out["rows"] == 2 * 64, out
    assert out["append_flips"] == 0, out
    assert out["max_iteration_diff"] <= 2, out
    assert out["max_explicit_residual_gpu"] <= out["tol"], out
    assert out["max_solution_reldiff"] <= 1e-6, out
    assert out["pass"], out
