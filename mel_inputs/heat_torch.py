"""Seeded synthetic-input generator on the GPU (bench plumbing, not the method):
the same exact implicit-Euler heat solutions as mel_inputs.heat (Eq. 2,
P:294-306; readings in that module), computed with dense DST-I matrices in fp64
torch so that the paper-shaped 1000x1000 basis (5 x 100 fields) takes well under a
second on a B200 instead of minutes on the host.  Holds none of the method's
arithmetic."""
from __future__ import annotations

import math

import torch


def basis(n: int, tau: int, device="cuda", alpha: float = 1.0, dt: float = 0.01, length: float = 1.0,
          out_dtype=torch.float32) -> torch.Tensor:
    """phi[c, t] = u^t for X = e_c, shape (5, tau, n*n) in out_dtype on `device`."""
    m = n - 2
    h = length / (n - 1)
    i = torch.arange(1, n - 1, dtype=torch.float64, device=device)
    S = math.sqrt(2.0 / (n - 1)) * torch.sin(math.pi * i[:, None] * i[None, :] / (n - 1))   # orthonormal DST-I
    lam = (4.0 / (h * h)) * torch.sin(i * math.pi / (2.0 * (n - 1))) ** 2
    denom = 1.0 + alpha * dt * (lam[:, None] + lam[None, :])
    c = alpha * dt / (h * h)
    phi = torch.empty((5, tau, n * n), dtype=out_dtype, device=device)
    for comp in range(5):
        X = [0.0] * 5
        X[comp] = 1.0
        t_ic, (tx1, ty1, tx2, ty2) = X[0], X[1:]
        bterm = torch.zeros((m, m), dtype=torch.float64, device=device)
        bterm[:, 0] += tx1; bterm[:, -1] += tx2; bterm[0, :] += ty1; bterm[-1, :] += ty2
        bterm *= c
        u = torch.full((m, m), t_ic, dtype=torch.float64, device=device)
        f = torch.empty((n, n), dtype=torch.float64, device=device)
        phi[comp, 0] = t_ic
        for t in range(1, tau):
            u = S @ ((S @ (u + bterm) @ S) / denom) @ S
            f[1:-1, 1:-1] = u
            f[1:-1, 0] = tx1; f[1:-1, -1] = tx2; f[0, 1:-1] = ty1; f[-1, 1:-1] = ty2
            f[0, 0] = 0.5 * (tx1 + ty1); f[0, -1] = 0.5 * (tx2 + ty1)
            f[-1, 0] = 0.5 * (tx1 + ty2); f[-1, -1] = 0.5 * (tx2 + ty2)
            phi[comp, t] = f.reshape(-1).to(out_dtype)
    return phi


def fields(phi: torch.Tensor, X: torch.Tensor, t: torch.Tensor) -> torch.Tensor:
    """u_X^t = sum_c X_c phi_c^t for a batch: X (k, 5) kelvin, t (k,) -> (k, n*n) fp32."""
    sel = phi[:, t, :]                                   # (5, k, N)
    return torch.einsum("kc,ckn->kn", X.to(sel.dtype), sel).contiguous()
