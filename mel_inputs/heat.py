"""Seeded synthetic-input generator: the 2D heat-equation client of the paper.

This module is an INPUT GENERATOR shared by the oracle tests and the bench.  It
holds none of the method's arithmetic (no reservoir, no MLP, no optimiser); it
only produces the time steps u_X^t that the simulation clients stream.

Paper anchors (section 4.1 "Equation and deep surrogate
architectures"):
  * Eq. 2: dT/dt = alpha * lap(T), T(x,y,0) = T_IC,
    T(0,y,t) = T_x1, T(L,y,t) = T_x2, T(x,0,t) = T_y1, T(x,L,t) = T_y2.
  * finite differences, implicit Euler, 1000x1000 grid, 100 time
    steps of dt = 0.01 s, alpha = 1 m^2/s.
  * X = (T_IC, T_x1, T_y1, T_x2, T_y2) sampled in [100, 500] K.
  * fields are converted from 64 to 32 bit before being sent.

Readings:
  * unit square, L = 1 m, h = L/(n-1), n nodes per axis including the boundary;
  * t = 0 emits T_IC at every node (boundary included);
  * t >= 1: edges carry their Dirichlet value, corners the mean of the two
    adjacent boundary values (corners are never read by the 5-point stencil);
  * the implicit system is solved exactly (not to a tolerance) by DST-I
    diagonalisation of the 5-point Laplacian.
Field layout: k = j*n + i, i = x index (column), j = y index (row).
"""
from __future__ import annotations

import numpy as np
import scipy.fft

ALPHA = 1.0
DT = 0.01
LENGTH = 1.0


def _eigs(n: int, length: float = LENGTH) -> np.ndarray:
    """1D eigenvalues of -L_h on the m = n-2 interior nodes (Dirichlet):
    lambda_p = (4/h^2) sin^2(p*pi/(2(n-1))), p = 1..n-2."""
    h = length / (n - 1)
    p = np.arange(1, n - 1, dtype=np.float64)
    return (4.0 / (h * h)) * np.sin(p * np.pi / (2.0 * (n - 1))) ** 2


def _dst2(a: np.ndarray) -> np.ndarray:
    # orthonormal DST-I along both axes; it is an involution (its own inverse)
    return scipy.fft.dstn(a, type=1, norm="ortho", workers=-1)


def boundary_terms(n: int, bc: tuple[float, float, float, float],
                   alpha: float = ALPHA, dt: float = DT, length: float = LENGTH) -> np.ndarray:
    """alpha*dt/h^2 * (sum of the Dirichlet neighbours) for every interior node.
    bc = (T_x1, T_y1, T_x2, T_y2) in the order of X."""
    tx1, ty1, tx2, ty2 = bc
    h = length / (n - 1)
    c = alpha * dt / (h * h)
    m = n - 2
    b = np.zeros((m, m), dtype=np.float64)  # [j-1, i-1]
    b[:, 0] += tx1       # i = 1 touches x = 0
    b[:, -1] += tx2      # i = n-2 touches x = L
    b[0, :] += ty1       # j = 1 touches y = 0
    b[-1, :] += ty2      # j = n-2 touches y = L
    return c * b


def implicit_euler_step(u_int: np.ndarray, bterm: np.ndarray, n: int,
                        alpha: float = ALPHA, dt: float = DT, length: float = LENGTH) -> np.ndarray:
    """One implicit-Euler step (I - alpha*dt*L_h) u^{t} = u^{t-1} + bterm, solved
    exactly by separable DST-I diagonalisation.  u_int is (n-2, n-2) [j, i]."""
    lam = _eigs(n, length)
    denom = 1.0 + alpha * dt * (lam[:, None] + lam[None, :])
    return _dst2(_dst2(u_int + bterm) / denom)


def assemble(u_int: np.ndarray, n: int, bc: tuple[float, float, float, float]) -> np.ndarray:
    """Full n*n field from the interior and the boundary values (t >= 1)."""
    tx1, ty1, tx2, ty2 = bc
    f = np.empty((n, n), dtype=np.float64)
    f[1:-1, 1:-1] = u_int
    f[1:-1, 0] = tx1
    f[1:-1, -1] = tx2
    f[0, 1:-1] = ty1
    f[-1, 1:-1] = ty2
    f[0, 0] = 0.5 * (tx1 + ty1)
    f[0, -1] = 0.5 * (tx2 + ty1)
    f[-1, 0] = 0.5 * (tx1 + ty2)
    f[-1, -1] = 0.5 * (tx2 + ty2)
    return f


def simulate(X, n: int, tau: int, alpha: float = ALPHA, dt: float = DT,
             length: float = LENGTH, dtype=np.float32) -> np.ndarray:
    """Run one client: returns the tau emitted fields u_X^t, t = 0..tau-1, as
    (tau, n*n) in `dtype` (fp32 = the paper's wire precision; the cast is
    round-to-nearest-even)."""
    X = np.asarray(X, dtype=np.float64)
    t_ic, bc = X[0], (X[1], X[2], X[3], X[4])
    out = np.empty((tau, n * n), dtype=np.float64)
    out[0] = t_ic
    u = np.full((n - 2, n - 2), t_ic, dtype=np.float64)
    bterm = boundary_terms(n, bc, alpha, dt, length)
    for t in range(1, tau):
        u = implicit_euler_step(u, bterm, n, alpha, dt, length)
        out[t] = assemble(u, n, bc).reshape(-1)
    return out.astype(dtype) if dtype is not None else out


def basis(n: int, tau: int, **kw) -> np.ndarray:
    """The map X -> u_X^t is linear (Eq. 2 with linear BC/IC data), so
    u_X^t = sum_c X_c * phi_c^t with phi_c the solution for X = e_c.
    Returns phi as fp64 (5, tau, n*n)."""
    return np.stack([simulate(np.eye(5)[c], n, tau, dtype=None, **kw) for c in range(5)])


def fields_from_basis(phi: np.ndarray, X, t) -> np.ndarray:
    """u_X^t from the fp64 basis, rounded to fp32."""
    X = np.asarray(X, dtype=np.float64)
    return np.tensordot(X, phi[:, t, :], axes=(0, 0)).astype(np.float32)
