"""Hybrid forward evaluator (paper_1602_00138_b200/inversion.py) against the
reference's HybridEvaluator contract (proj/src/inversion.cpp:53-106,
proj/tests/test_inversion.cpp): the first K_* distinct points go through the
basis builder and their own solutions serve transfer / Jacobian, the next new
point switches to the reduced model on V, a full-order request after the
switch is a SolverError; counters as in the reference."""
import numpy as np
import pytest

from paper_1602_00138_b200 import problem as P


def test_absorption_supports_match_finite_differences():
    from paper_1602_00138_b200 import inversion as I
    c = P.CONFIGS["T3"]
    g = c.grid
    p = c.point_params(1)
    v = I.params_to_vector(p)
    sup = I.absorption_supports(g, p)
    assert len(sup) == v.size
    for k in range(v.size):
        e = np.zeros(v.size)
        e[k] = 1e-6
        fd = (P.absorption(g, I.vector_to_params(v + e, c.m_rbf, c.d))
              - P.absorption(g, I.vector_to_params(v - e, c.m_rbf, c.d))) / 2e-6
        dense = np.zeros(g.n)
        ix, w = sup[k]
        dense[ix] = w
        assert np.abs(dense - fd).max() <= 1e-6 * max(1e-12, np.abs(fd).max()) + 1e-9


def test_clamp_and_vector_roundtrip():
    from paper_1602_00138_b200 import inversion as I
    c = P.CONFIGS["T3"]
    p = c.point_params(2)
    v = I.params_to_vector(p)
    q = I.vector_to_params(v, c.m_rbf, c.d)
    assert np.array_equal(q.centres, p.centres) and np.array_equal(q.widths, p.widths)
    v[-1] = -3.0
    assert I.clamp_widths(v, c.m_rbf, c.d)[-1] == 1e-6


@pytest.mark.gpu
def test_hybrid_evaluator_switches_to_rom():
    from paper_1602_00138_b200 import build
    build.build()
    from paper_1602_00138_b200 import inversion as I, romdot as R
    c = P.CONFIGS["T3c"]
    g, lay = c.grid, c.layout()
    w = 0.1
    f0 = c.fields(0, w)
    lam, U0 = R.smallest_eigenpairs(R.SchurOperator(g, c.fields(0), np.float64), c.k, 1e-8)
    X0, _ = R.initial_solutions(R.SchurOperator(g, f0, c.dtype), lay, c.tol)
    pts = [I.params_to_vector(c.point_params(i)) for i in range(5)]
    ev = I.HybridEvaluator(c, U0, X0, pts[0], k_systems=2, tol_basis=c.tol, omega=w)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731

    def fom(v):
        return R.fom_transfer(R.SchurOperator(g, ev.fields(v), c.dtype), lay, 1e-12)[0]

    psi0 = ev.transfer(pts[0])  # served by the seed's X0, no system
    assert ev.systems_used == 0 and ev.function_evals == 1
    assert rel(psi0, fom(pts[0])) <= 1e-6
    psi1 = ev.transfer(pts[1])
    assert ev.systems_used == 1 and not ev.in_rom_mode
    assert rel(psi1, fom(pts[1])) <= 1e-6
    J1 = ev.jacobian(pts[1])  # the same point: cached solutions, no new system
    assert ev.systems_used == 1 and ev.jacobian_evals == 1
    sup = I.absorption_supports(g, I.vector_to_params(pts[1], c.m_rbf, c.d))
    Jf = R.fom_jacobian(R.SchurOperator(g, ev.fields(pts[1]), c.dtype), lay, sup, -g.h ** 2, 1e-12)
    assert rel(J1, Jf) <= 1e-6
    ev.transfer(pts[2])
    assert ev.systems_used == 2 and len(ev.visited) == 3 and len(ev.build_log) == 2 * lay.n_rhs
    psi3 = ev.transfer(pts[3])  # K_* = 2 systems used: switch to the ROM on V
    assert ev.in_rom_mode and ev.systems_used == 2
    assert rel(psi3, fom(pts[3])) <= 1e-3, rel(psi3, fom(pts[3]))
    J3 = ev.jacobian(pts[3])
    assert np.isfinite(J3).all() and J3.shape == J1.shape
    with pytest.raises(R.SolverError):
        ev.solutions_for(pts[4])
    assert ev.full_order_solves == lay.n_rhs + ev.appends
