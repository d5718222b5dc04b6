"""Shared test fixtures: the reference's desk problems (test_basis.cpp:16-53)
and the ROM observables of rom.cpp:9-35 used by the parity protocol."""
import numpy as np

import oracle as orc
from paper_1602_00138_b200 import problem as P


class Desk:
    """Reference 2D desk problem: [0,4]^2, D0 = 0.3, nx = ny = n."""

    def __init__(self, n, n_src, n_det):
        self.grid = P.GridSpec.reference_2d(n, n)
        self.layout = P.make_layout(self.grid, (n_src,), (n_det,), src_high=True)
        self.B = self.layout.dense(self.grid.n)
        self.h2 = self.grid.h ** 2
        self.x = self.grid.coordinates()

    def mu_of(self, offset):
        # smooth 4-bump absorption standing in for the PaLS desk params (test_basis.cpp:33-43)
        c = np.array([[1.0, 1.0], [3.0, 1.0], [1.0, 3.0], [3.0, 3.0]])
        phi = np.full(self.grid.n, -0.5)
        for j in range(4):
            r = np.linalg.norm(self.x - c[j], axis=1) / (0.9 + offset * (1 + j))
            phi += np.where(r < 3, np.exp(-0.5 * r * r), 0.0)
        return self.h2 * (0.01 + 0.02 * P.smooth_heaviside(phi))

    def op(self, offset, dtype=np.float64):
        return orc.Operator.grid(self.grid, P.constant_fields(self.grid, self.mu_of(offset)), dtype)

    def A(self, offset):
        return self.op(offset).matrix()


def rom_transfer(V, A, B, C):
    """Psi_r = C_r^T A_r^-1 B_r with one-sided (bilinear) projection (rom.cpp:9-35)."""
    Ar = V.T @ (A @ V)
    Ar = 0.5 * (Ar + Ar.T)
    return (C.T @ V) @ np.linalg.solve(Ar, V.T @ B)


def rom_jacobian(V, A, B, C, directions):
    """d Psi_r / d mu along diagonal directions: -C_r^T A_r^-1 (V^T diag(dk) V) A_r^-1 B_r."""
    Ar = V.T @ (A @ V)
    Ar = 0.5 * (Ar + Ar.T)
    Y = np.linalg.solve(Ar, V.T @ B)
    Z = np.linalg.solve(Ar.T, V.T @ C)
    return np.stack([-(Z.T @ (V.T @ (dk[:, None] * V)) @ Y).ravel() for dk in directions], axis=1)


def fom_transfer(A, B, C):
    return C.T @ np.linalg.solve(A, B)
