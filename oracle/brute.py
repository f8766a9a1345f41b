"""Brute-force numpy tier of the oracle (grids <= 16x16).  TEST INFRASTRUCTURE ONLY.

Assembles each filter's N x N periodic convolution matrix K_i explicitly
("K_i is an N x N highly sparse matrix, implemented as 2D
convolution of the image u with filter kernel k_i") and evaluates the energy,
gradient and Hessian with dense linear algebra.  Used to validate the C oracle's
indexing; the C oracle and this tier are pinned independently in
tests/test_oracle_pins.py (scipy convolution, finite differences, closed forms).
"""
from __future__ import annotations

import numpy as np


def conv_matrix(k: np.ndarray, H: int, W: int) -> np.ndarray:
    """Dense K with (K u)[y,x] = sum_{a,b} k[a,b] u[(y-a+c) % H, (x-b+c) % W] (R-2, R-3)."""
    k = np.asarray(k, np.float64)
    m = k.shape[0]
    c = (m - 1) // 2
    N = H * W
    K = np.zeros((N, N))
    for y in range(H):
        for x in range(W):
            p = y * W + x
            for a in range(m):
                for b in range(m):
                    q = ((y - a + c) % H) * W + ((x - b + c) % W)
                    K[p, q] += k[a, b]
    return K


def energy_grad_w(w, filters, theta):
    """F(w) = sum_i theta_i sum_p log(1 + (K_i e^w)_p^2); grad = diag(e^w) sum theta_i K_i^T rho'."""
    w = np.asarray(w, np.float64)
    H, W = w.shape
    u = np.exp(w).ravel()
    F = 0.0
    g = np.zeros(H * W)
    for k, th in zip(filters, theta):
        K = conv_matrix(k, H, W)
        r = K @ u
        F += float(th) * np.sum(np.log1p(r * r))
        g += float(th) * (K.T @ (2 * r / (1 + r * r)))
    return F, (u * g).reshape(H, W)


def hessian_w(w, filters, theta) -> np.ndarray:
    """Dense Hessian of F(w) = E_FoE(e^w): diag(u*s) + diag(u) [sum theta K^T diag(rho'') K] diag(u)."""
    w = np.asarray(w, np.float64)
    H, W = w.shape
    u = np.exp(w).ravel()
    N = H * W
    s = np.zeros(N)
    M = np.zeros((N, N))
    for k, th in zip(filters, theta):
        K = conv_matrix(k, H, W)
        r = K @ u
        s += float(th) * (K.T @ (2 * r / (1 + r * r)))
        rpp = 2 * (1 - r * r) / (1 + r * r) ** 2
        M += float(th) * (K.T @ (rpp[:, None] * K))
    return np.diag(u * s) + u[:, None] * M * u[None, :]


def prox_bisect(what, ft, tau, l1, l2, iters=200):
    """Root of phi(z) = z - what + tau[l1(1 - f^2 e^{-2z}) + l2(e^{2z} - f^2)] by pure bisection."""
    lf = np.log(ft)
    lo, hi = min(what, lf) - 1.0, max(what, lf) + 1.0

    def phi(z):
        return z - what + tau * (l1 * (1 - ft * ft * np.exp(-2 * z)) + l2 * (np.exp(2 * z) - ft * ft))

    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if phi(mid) > 0:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def hessian_u(u, filters, theta) -> np.ndarray:
    """Dense Hessian of F(u) = E_FoE(u) (model (6)): sum_i theta_i K_i^T diag(rho''(K_i u)) K_i."""
    u = np.asarray(u, np.float64)
    H, W = u.shape
    x = u.ravel()
    M = np.zeros((H * W, H * W))
    for k, th in zip(filters, theta):
        K = conv_matrix(k, H, W)
        r = K @ x
        rpp = 2 * (1 - r * r) / (1 + r * r) ** 2
        M += float(th) * (K.T @ (rpp[:, None] * K))
    return M
