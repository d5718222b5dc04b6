"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py
with the CPU oracle): the oracle must reproduce them exactly (determinism,
independent of thread count), and the CUDA path must match them within the
parity tolerances (App. C): +-2 iterations and identical append flags per
BuildLog row, reduced transfer within 1e-8."""
import os

import numpy as np
import pytest

import oracle as orc
from helpers import rom_transfer
from paper_1602_00138_b200 import problem as P

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["T2", "T3c"]


def load(name):
    return np.load(os.path.join(HERE, f"{name}.npz"))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name):
    z = load(name)
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    gb = orc.GlobalBasis(z["U0"], z["X0"], c.cap)
    logs = []
    op = None
    for s, (pt, w) in enumerate(c.systems(), start=1):
        op = orc.Operator.grid(g, c.fields(pt, w), c.dtype)
        pr = orc.process_system(gb, op, lay, c.tol, s)
        logs += [[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in pr.log]
    logs = np.array(logs)
    gl = z["log"]
    assert np.array_equal(logs[:, [0, 1, 3, 4]], gl[:, [0, 1, 3, 4]])
    assert np.allclose(logs[:, 2], gl[:, 2], rtol=1e-12, atol=0)
    assert gb.cols == int(z["cols"])
    B = lay.dense(g.n, c.dtype)
    psi = rom_transfer(gb.V, op.matrix(), B[:, : lay.n_src], B[:, lay.n_src:])
    assert np.allclose(psi, z["psi"], rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_build_matches_golden(name):
    from paper_1602_00138_b200 import build, romdot as R
    build.build()
    z = load(name)
    c = P.CONFIGS[name]
    g, lay = c.grid, c.layout()
    gb = R.GlobalBasis(z["U0"], z["X0"], c.cap)
    logs = []
    for s, (pt, w) in enumerate(c.systems(), start=1):
        pr = R.process_system(gb, R.SchurOperator(g, c.fields(pt, w), c.dtype), lay, c.tol, s, want_X=False)
        logs += [[r.system, r.rhs, r.init_relres, r.iterations, float(r.appended)] for r in pr.log]
    logs = np.array(logs)
    gl = z["log"]
    assert np.array_equal(logs[:, 4], gl[:, 4])
    assert np.all(np.abs(logs[:, 3] - gl[:, 3]) <= 2)
    assert gb.cols == int(z["cols"])
    pt, w = c.systems()[-1]
    A = orc.Operator.grid(g, c.fields(pt, w), c.dtype).matrix()
    B = lay.dense(g.n, c.dtype)
    psi = rom_transfer(gb.V, A, B[:, : lay.n_src], B[:, lay.n_src:])
    assert np.linalg.norm(psi - z["psi"]) <= 1e-8 * np.linalg.norm(z["psi"])
