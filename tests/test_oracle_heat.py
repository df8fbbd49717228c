"""Pins for the heat-equation input generator (mel_inputs/heat.py), PAPER.md
Eq. 2 and P:304 (implicit Euler FD): closed forms, invariants and a
textbook dense solve."""
import numpy as np
import pytest

from mel_inputs import heat


def test_discrete_eigenmode_decays_by_exact_factor():
    # interior sin(p pi x) sin(q pi y) with zero BCs is an eigenvector of the
    # 5-point Laplacian; one implicit step multiplies it by 1/(1 + a dt lam_pq).
    n, p, q = 9, 2, 3
    h = 1.0 / (n - 1)
    x = np.arange(1, n - 1) * h
    u0 = np.outer(np.sin(q * np.pi * x), np.sin(p * np.pi * x))  # [j, i]
    lam = (4 / h**2) * (np.sin(p * np.pi * h / 2) ** 2 + np.sin(q * np.pi * h / 2) ** 2)
    u1 = heat.implicit_euler_step(u0, np.zeros_like(u0), n)
    np.testing.assert_allclose(u1, u0 / (1 + heat.ALPHA * heat.DT * lam), atol=1e-15, rtol=0)


def _dense_step(u_int, bterm, n):
    m = n - 2
    h = 1.0 / (n - 1)
    c = heat.ALPHA * heat.DT / h**2
    A = np.zeros((m * m, m * m))
    for j in range(m):
        for i in range(m):
            k = j * m + i
            A[k, k] = 1 + 4 * c
            for (jj, ii) in ((j - 1, i), (j + 1, i), (j, i - 1), (j, i + 1)):
                if 0 <= jj < m and 0 <= ii < m:
                    A[k, jj * m + ii] = -c
    return np.linalg.solve(A, (u_int + bterm).reshape(-1)).reshape(m, m)


@pytest.mark.parametrize("n", [4, 5, 6])
def test_matches_dense_linear_solve(n):
    rng = np.random.default_rng(n)
    X = rng.uniform(100, 500, 5)
    u = np.full((n - 2, n - 2), X[0])
    bterm = heat.boundary_terms(n, tuple(X[1:]))
    for _ in range(3):
        ref = _dense_step(u, bterm, n)
        u = heat.implicit_euler_step(u, bterm, n)
        np.testing.assert_allclose(u, ref, rtol=1e-12, atol=0)


def test_constant_field_is_fixed_point():
    f = heat.simulate([300.0] * 5, 8, 5, dtype=None)
    np.testing.assert_allclose(f, 300.0, rtol=0, atol=1e-12)


def test_maximum_principle():
    rng = np.random.default_rng(0)
    for _ in range(30):
        X = rng.uniform(100, 500, 5)
        f = heat.simulate(X, 9, 6, dtype=None)
        assert f.min() >= X.min() - 1e-9 and f.max() <= X.max() + 1e-9


@pytest.mark.parametrize("n", [9, 10])
def test_steady_state_centre_is_mean_of_boundaries(n):
    # superposition of the four rotated one-hot-side problems on a square grid
    X = np.array([123.0, 100.0, 200.0, 340.0, 600.0])
    f = heat.simulate(X, n, 400, dtype=None)[-1].reshape(n, n)
    c = (n - 1) // 2
    centre = f[c, c] if n % 2 else f[c:c + 2, c:c + 2].mean()
    assert abs(centre - X[1:].mean()) < 1e-9


def test_linearity_and_basis_superposition():
    rng = np.random.default_rng(3)
    X1, X2 = rng.uniform(100, 500, 5), rng.uniform(100, 500, 5)
    a = heat.simulate(X1 + X2, 7, 4, dtype=None)
    b = heat.simulate(X1, 7, 4, dtype=None) + heat.simulate(X2, 7, 4, dtype=None)
    np.testing.assert_allclose(a, b, rtol=1e-12)
    phi = heat.basis(7, 4)
    for t in range(4):
        np.testing.assert_allclose(heat.fields_from_basis(phi, X1, t),
                                   heat.simulate(X1, 7, 4)[t], rtol=1e-6)


def test_t0_emits_initial_condition_everywhere_and_tau_steps():
    f = heat.simulate([250.0, 100, 200, 300, 400], 6, 10)
    assert f.shape == (10, 36) and f.dtype == np.float32
    assert np.all(f[0] == np.float32(250.0))
    g = f[1].reshape(6, 6)
    assert np.all(g[1:-1, 0] == 100) and np.all(g[1:-1, -1] == 300)
    assert np.all(g[0, 1:-1] == 200) and np.all(g[-1, 1:-1] == 400)


def test_torch_generator_matches_numpy_generator():
    import torch
    from mel_inputs import heat_torch
    phi_t = heat_torch.basis(9, 5, device="cpu", out_dtype=torch.float64).numpy()
    phi_n = heat.basis(9, 5)
    np.testing.assert_allclose(phi_t, phi_n, rtol=1e-11, atol=1e-12)
