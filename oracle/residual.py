"""Accuracy metrics.  ORACLE / TEST INFRASTRUCTURE ONLY.

Eq. 14 prints R_i = ||A u_i - sigma_i v_i|| / sigma_i, which is
dimensionally inconsistent for m != n; read as ||A v_i - sigma_i u_i||_2
(reading R13).  Returned both sigma_i-relative (the paper's R_i) and
sigma_1-relative (the north_star's e_i).
Eckart-Young (Eq. 3): ||A - U_r S_r V_r^T||_2 ~ sigma_{r+1},
estimated by power iteration on the implicit operator.
"""
from __future__ import annotations

import numpy as np


def residuals(op, U, S, V):
    """Returns (e, R): e_i = ||A v_i - s_i u_i|| / s_1, R_i = ... / s_i."""
    res = op.matmul(V) - U * S[None, :]
    nr = np.linalg.norm(res, axis=0)
    return nr / S[0], nr / np.where(S > 0, S, 1.0)


def eckart_young_2norm(op, U, S, V, iters: int = 300, seed: int = 7):
    """||A - U S V^T||_2 by power iteration on E^T E (E implicit)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(op.n)
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = op.matmul(x[:, None])[:, 0] - U @ (S * (V.T @ x))
        z = op.rmatmul(y[:, None])[:, 0] - V @ (S * (U.T @ y))
        lam = np.linalg.norm(z)
        x = z / lam
    return float(np.sqrt(lam))
