"""ORACLE (test infrastructure only -- never imported by the product path).

The direct deep surrogate f_theta(X, t) ~ u_X^t and its
training step, in plain fp64 numpy, in the paper's order:

  * architecture: input 6 = (X normalised, t normalised), hidden layers
    with ReLU (2 x 256 in the paper; 1 x 32 for the tiny config), linear output of
    N = n*n neurons.
  * loss: MSE ("Min. MSE"), mean over batch and outputs:
        L = sum_{b,n} (Y - T)^2 / (B * N)
  * forward and backward passes, ReLU'(0) = 0 (reading Q25).
  * Adam, lr0 = 1e-3, (beta1, beta2, eps) = (0.9, 0.999, 1e-8) (reading
    Q23), bias-corrected PyTorch form, no weight decay.
  * LR schedule ("halved every 1000 batches", "every 10,000 training
    samples ... minimum of 2.5E-4"; reading Q24: counted in global samples
    consumed before the step, repeats included):
        lr_k = max(2.5e-4, 1e-3 * 2^-floor(S_k / 10^4))
  * normalisation (reading Q13): xn = ((X_c - 100)/400, t/tau), targets = the
    reservoir's stored values (see oracle.reservoir) promoted to fp64.
  * init (reading Q22): W, b ~ U(-a, a), a = 1/sqrt(fan_in) (PyTorch nn.Linear
    range), drawn from the Philox INIT stream, computed in fp64, rounded to fp32.
"""
from __future__ import annotations

import numpy as np

from . import philox

BETA1, BETA2, EPS = 0.9, 0.999, 1e-8
LR0, LR_MIN, LR_HALVING = 1e-3, 2.5e-4, 10000


def layer_dims(n_field: int, hidden) -> list[int]:
    return [6] + [int(h) for h in hidden if h] + [int(n_field)]


def n_params(dims) -> int:
    return sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))


def init_params(dims, seed: int):
    """Philox INIT stream: tensor ids 2l (W_l, row-major [out][in]) and 2l+1 (b_l),
    element index = counter.  Returns fp32 arrays."""
    params = []
    for l in range(len(dims) - 1):
        fan_in, fan_out = dims[l], dims[l + 1]
        a = 1.0 / np.sqrt(np.float64(fan_in))
        out = []
        for tid, count in ((2 * l, fan_out * fan_in), (2 * l + 1, fan_out)):
            u = philox.unit_double(philox.r64(seed, philox.TAG_INIT, np.arange(count, dtype=np.uint64), tid))
            out.append(((2.0 * u - 1.0) * a).astype(np.float32))
        params.append((out[0].reshape(fan_out, fan_in), out[1]))
    return params


def normalise_inputs(X_f32, t, tau: int) -> np.ndarray:
    X = np.asarray(X_f32, dtype=np.float32).astype(np.float64)
    t = np.asarray(t, dtype=np.float64)
    return np.concatenate([(X - 100.0) / 400.0, (t / tau)[:, None]], axis=1)


def forward(params, xn):
    """Returns the list of pre-activations Z_l and activations H_l (H_0 = xn)."""
    H = [np.asarray(xn, dtype=np.float64)]
    Z = []
    L = len(params)
    for l, (W, b) in enumerate(params):
        z = H[-1] @ np.asarray(W, np.float64).T + np.asarray(b, np.float64)
        Z.append(z)
        H.append(np.maximum(z, 0.0) if l < L - 1 else z)
    return Z, H


def sse_and_grads(params, xn, tn):
    """Raw sum of squared errors S = sum (Y - T)^2 and its exact gradient dS/dtheta
    by reverse mode.  The mean-loss gradient is this / (B*N) (or / (N*sum n_r) in
    the data-parallel case, oracle.trainer)."""
    Z, H = forward(params, xn)
    Y = H[-1]
    R = Y - np.asarray(tn, dtype=np.float64)
    S = float(np.sum(R * R))
    grads = [None] * len(params)
    dZ = 2.0 * R                                   # dS/dY (output is linear)
    for l in range(len(params) - 1, -1, -1):
        W = np.asarray(params[l][0], np.float64)
        grads[l] = (dZ.T @ H[l], dZ.sum(axis=0))   # dW = dZ^T H_{l}, db = sum_b dZ
        if l > 0:
            dH = dZ @ W
            dZ = dH * (Z[l - 1] > 0.0)             # ReLU'(0) = 0
    return S, grads


def mse(params, xn, tn) -> float:
    _, H = forward(params, xn)
    R = H[-1] - np.asarray(tn, dtype=np.float64)
    return float(np.mean(R * R))


def loss_and_grads(params, xn, tn):
    S, g = sse_and_grads(params, xn, tn)
    denom = float(np.asarray(tn).size)
    return S / denom, [(dW / denom, db / denom) for dW, db in g]


def lr_schedule(samples_before: int, lr0=LR0, lr_min=LR_MIN, interval=LR_HALVING) -> float:
    return max(lr_min, lr0 * 2.0 ** (-(int(samples_before) // int(interval))))


def adam_update(p, g, m, v, k: int, lr: float, beta1=BETA1, beta2=BETA2, eps=EPS):
    """One Adam update of one tensor at 1-based step k (fp64):
        m <- b1 m + (1-b1) g ;  v <- b2 v + (1-b2) g^2
        p <- p - lr * (m / (1-b1^k)) / (sqrt(v / (1-b2^k)) + eps)"""
    g = np.asarray(g, np.float64)
    m = beta1 * np.asarray(m, np.float64) + (1.0 - beta1) * g
    v = beta2 * np.asarray(v, np.float64) + (1.0 - beta2) * g * g
    p = np.asarray(p, np.float64) - lr * (m / (1.0 - beta1 ** k)) / (np.sqrt(v / (1.0 - beta2 ** k)) + eps)
    return p, m, v


class Adam:
    """Adam (Kingma & Ba), bias-corrected, fp64 state; tensors in the flat order
    W_1, b_1, W_2, b_2, ... (tensor id = index)."""

    def __init__(self, tensors):
        self.m = [np.zeros(np.shape(x), np.float64) for x in tensors]
        self.v = [np.zeros(np.shape(x), np.float64) for x in tensors]
        self.k = 0

    def step(self, tensors, grads, lr: float):
        self.k += 1
        out = []
        for i, (p, g) in enumerate(zip(tensors, grads)):
            p, self.m[i], self.v[i] = adam_update(p, g, self.m[i], self.v[i], self.k, lr)
            out.append(p)
        return out


def flatten(params):
    return [x for Wb in params for x in Wb]


def unflatten(tensors):
    return [(tensors[2 * i], tensors[2 * i + 1]) for i in range(len(tensors) // 2)]
