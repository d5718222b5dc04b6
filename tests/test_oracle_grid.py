"""Oracle operator pinned to the reference's grid tests (test_grid.cpp,
acceptance.cpp criterion 1): the eliminated-Robin Schur operator must give the
same transfer function as the unreduced block system assembled exactly as
grid.cpp:38-84 does, and be SPD."""
import numpy as np
import pytest

import oracle as orc
from paper_1602_00138_b200 import problem as P


def reference_blocks(nx, ny, h, d0, A):
    """Dense restatement of assemble_blocks (grid.cpp:38-84), boundary-first."""
    nb, ni = 2 * nx, (ny - 2) * nx
    robin = 2.0 * A * d0 / h
    G = np.diag(np.full(nb, 1.0 + robin))
    D1 = np.zeros((nb, ni))
    D2 = np.zeros((ni, nb))
    L = np.zeros((ni, ni))
    idx = lambda i, j: (j - 1) * nx + i
    for i in range(nx):
        bb, tb = i, nx + i
        pb, pt = idx(i, 1), idx(i, ny - 2)
        D1[bb, pb] = -robin
        D1[tb, pt] = -robin
        D2[pb, bb] = -d0
        D2[pt, tb] = -d0
    for j in range(1, ny - 1):
        for i in range(nx):
            p = idx(i, j)
            L[p, p] = 4.0 * d0
            if i > 0: L[p, idx(i - 1, j)] = -d0
            if i < nx - 1: L[p, idx(i + 1, j)] = -d0
            if j > 1: L[p, idx(i, j - 1)] = -d0
            if j < ny - 2: L[p, idx(i, j + 1)] = -d0
    return G, D1, D2, L


@pytest.mark.parametrize("n", [5, 7, 9, 12])
def test_schur_matches_dense_block_transfer(n):
    # acceptance.cpp:113-140 / test_grid.cpp:78-99
    rng = np.random.default_rng(42 + n)
    g = P.GridSpec.reference_2d(n, n, b1=1.0)
    G, D1, D2, L = reference_blocks(n, n, g.h, g.D_bg, g.A)
    lay = P.make_layout(g, (2,), (3,), src_high=True)
    nb = 2 * n
    src = P.evenly_spaced_positions(n, 2)
    det = P.evenly_spaced_positions(n, 3)
    B1 = np.zeros((nb, 2)); C1 = np.zeros((nb, 3))
    for s, i in enumerate(src): B1[n + i, s] = 1.0      # top boundary nodes
    for t, i in enumerate(det): C1[i, t] = 1.0          # bottom boundary nodes
    worst = 0.0
    for trial in range(20):
        mu = g.h ** 2 * rng.uniform(size=g.n)
        full = np.block([[G, D1], [D2, L + np.diag(mu)]])
        rhs = np.vstack([B1, np.zeros((g.n, 2))])
        sol = np.linalg.solve(full, rhs)
        psi_full = C1.T @ sol[:nb]
        op = orc.Operator.grid(g, P.constant_fields(g, mu))
        A = op.matrix()
        B = lay.dense(g.n)
        X = np.linalg.solve(A, B[:, :2])
        psi = B[:, 2:].T @ X
        worst = max(worst, np.linalg.norm(psi - psi_full) / np.linalg.norm(psi_full))
        # Schur complement identity, entrywise
        S = L - D2 @ np.diag(1.0 / np.diag(G)) @ D1 + np.diag(mu)
        assert np.abs(A - S).max() <= 1e-14 * np.abs(S).max()
    assert worst <= 1e-10


def test_operator_spd_and_symmetric():
    g = P.GridSpec(d=3, N=(5, 6, 7), h=0.1, D_bg=0.33)
    rng = np.random.default_rng(1)
    f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=g.h ** 2 * rng.uniform(0.005, 0.05, g.n), shift=0.0)
    A = orc.Operator.grid(g, f).matrix()
    assert np.allclose(A, A.T, atol=0, rtol=1e-15)
    assert np.linalg.eigvalsh(A).min() > 0
    # complex shift: complex symmetric, A = A_real + i shift I
    fc = P.Fields(D=f.D, mu=f.mu, shift=0.02)
    Ac = orc.Operator.grid(g, fc, np.complex128).matrix()
    assert np.allclose(Ac, Ac.T, rtol=1e-15, atol=0)
    assert np.allclose(Ac.imag, 0.02 * np.eye(g.n))
    assert np.allclose(Ac.real, A)


def test_variable_d_stencil_formula():
    """Row p: diag = sum of face D (harmonic means / ghost D_p / Robin face) + mu."""
    g = P.GridSpec(d=2, N=(4, 5), h=0.25, D_bg=0.3)
    rng = np.random.default_rng(2)
    f = P.Fields(D=rng.uniform(0.3, 0.4, g.n), mu=rng.uniform(0, 0.01, g.n), shift=0.0)
    A = orc.Operator.grid(g, f).matrix()
    hm = lambda a, b: 2 * a * b / (a + b)
    for j in range(5):
        for i in range(4):
            p = g.node(i, j)
            diag = f.mu[p]
            for (di, dj) in [(-1, 0), (1, 0), (0, -1), (0, 1)]:
                ii, jj = i + di, j + dj
                if 0 <= ii < 4 and 0 <= jj < 5:
                    q = g.node(ii, jj)
                    assert A[p, q] == pytest.approx(-hm(f.D[p], f.D[q]), rel=1e-15)
                    diag += hm(f.D[p], f.D[q])
                elif dj != 0:
                    diag += g.robin_face
                else:
                    diag += f.D[p]
            assert A[p, p] == pytest.approx(diag, rel=1e-14)


def test_layout_single_nonzero_and_sign():
    g = P.GridSpec.reference_2d(15, 15)
    lay = P.make_layout(g, (3,), (3,), src_high=True)
    B = lay.dense(g.n)
    assert (np.count_nonzero(B, axis=0) == 1).all()
    assert (lay.val < 0).all()
    # Psi = C~^T A^-1 B~ > 0 (test_harness.cpp:140)
    mu = g.h ** 2 * np.full(g.n, 0.01)
    A = orc.Operator.grid(g, P.constant_fields(g, mu)).matrix()
    psi = B[:, 3:].T @ np.linalg.solve(A, B[:, :3])
    assert (psi > 0).all()


def test_normal_stream_python_matches_c():
    for seed in [0, 1, 77, 1234, 20160200 + 1000003]:
        s = P.NormalStream(seed)
        py = np.array([s.next() for _ in range(101)])
        c = orc.normal_stream(seed, 101)
        assert np.array_equal(py, c)


def test_evenly_spaced_positions():
    # grid.cpp:107-121 semantics
    assert P.evenly_spaced_positions(15, 3) == [1, 7, 13]
    assert P.evenly_spaced_positions(41, 1) == [20]
    assert P.evenly_spaced_positions(129, 16)[0] == 1 and P.evenly_spaced_positions(129, 16)[-1] == 127
    with pytest.raises(ValueError):
        P.evenly_spaced_positions(5, 4)
