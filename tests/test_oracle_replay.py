"""The checker's single-RHS replay (orc.replay_rhs, used by the C4
checkpoint-replay lockstep of oracle/replay.py) reproduces the checker's own
process_system (proj/src/basis.cpp:157-207) row by row, bitwise: the same
init_relres, iterations, append decision and solution X_j when each RHS is
replayed from the state the loop body starts it from (record-then-replay,
proj/tests/acceptance.cpp:201-250)."""
import numpy as np
import pytest

import oracle as orc
from paper_1602_00138_b200 import problem as P


def seed(c):
    g, lay = c.grid, c.layout()
    f0 = c.fields(0)
    _, U0 = orc.smallest_eigenpairs(orc.Operator.grid(g, f0), c.k, 1e-8)
    X0, _ = orc.initial_solutions(orc.Operator.grid(g, f0, c.dtype), lay, c.tol)
    return U0.astype(c.dtype), X0


@pytest.mark.parametrize("name", ["T2", "T3c"])
def test_replay_reproduces_process_system(name):
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    U0, X0 = seed(c)
    ref = orc.GlobalBasis(U0, X0, c.cap)
    gb = orc.GlobalBasis(U0, X0, c.cap)
    spaces = [gb.space(j) for j in range(lay.n_rhs)]  # PerRhsSpaces, grown by this test's appends
    for s, (pt, w) in enumerate(c.systems(), start=1):
        op = orc.Operator.grid(g, c.fields(pt, w), c.dtype)
        po = orc.process_system(ref, op, lay, c.tol, s)
        gb.refresh(op)
        for j in range(lay.n_rhs):
            rr = orc.replay_rhs(op, gb.V, gb.K_img, gb.R, spaces[j], lay.idx[j], lay.val[j], c.tol, c.cap,
                                want_y=True)
            row = po.log[j]
            assert rr.init_relres == row.init_relres
            assert rr.iterations == row.iterations
            assert rr.appended == row.appended
            assert np.array_equal(rr.X, po.X[:, j])
            if rr.appended:  # apply the decision the replay made (process_system's own append)
                assert gb.append(rr.y, op.apply(rr.y))
                spaces[j].append(gb.cols - 1)
        assert gb.cols == ref.cols
        assert np.array_equal(gb.V, ref.V)
        assert spaces == [ref.space(j) for j in range(lay.n_rhs)]


def test_replay_rejects_bad_inputs():
    c = P.CONFIGS["T2"]
    g, lay = c.grid, c.layout()
    U0, X0 = seed(c)
    gb = orc.GlobalBasis(U0, X0, c.cap)
    op = orc.Operator.grid(g, c.fields(1), c.dtype)
    gb.refresh(op)
    with pytest.raises(orc.ConfigError):
        orc.replay_rhs(op, gb.V, gb.K_img, gb.R, [0, gb.cols + 3], lay.idx[0], lay.val[0], c.tol)
    with pytest.raises(orc.ConfigError):
        orc.replay_rhs(op, gb.V, gb.K_img, gb.R, gb.space(0), g.n + 1, 1.0, c.tol)
    with pytest.raises(ValueError):
        orc.replay_rhs(op, np.ascontiguousarray(gb.V), gb.K_img, gb.R, gb.space(0), lay.idx[0], lay.val[0], c.tol)
