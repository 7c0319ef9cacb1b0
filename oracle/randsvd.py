"""RandSVD: truncated SVD via randomized subspace iteration.  Alg. 1
(P:66-92), Sec. 2.1.

ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation (reading R6): the paper's subspace width "r" is
l = r + p (p = oversampling), the paper's loop count "p" is q + 1
(q = power iterations; q = 0 is the direct method of [13]).  The start
block Q_0 is Gaussian and not orthonormalised (reading R10).  The QR
factorisations are Alg. 3 CGS-QR with panels of b_qr columns.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import DrawCtx, cgs_qr, small_svd, sign_normalize
from .philox import gaussian_block


@dataclass
class RandResult:
    U: np.ndarray
    S: np.ndarray
    V: np.ndarray
    R: np.ndarray
    Qbar: np.ndarray
    Q: np.ndarray


def randsvd(op, r: int, p: int, q: int, b_qr: int, seed: int,
            start=None) -> RandResult:
    m, n = op.m, op.n
    l = r + p
    assert m >= n and 1 <= r and l <= n and q >= 0 and b_qr >= 1
    ctx = DrawCtx(seed)
    Q = gaussian_block(n, l, seed, draw=0) if start is None else np.array(start, dtype=np.float64)
    for _ in range(q + 1):                       # j = 1..p  (p = q+1)
        Yb = op.matmul(Q)                        # S1
        Qb, _ = cgs_qr(Yb, b_qr, ctx)            # S2
        Y = op.rmatmul(Qb)                       # S3
        Q, R = cgs_qr(Y, b_qr, ctx)              # S4
    Ub, S, Vb = small_svd(R)                     # S5  R_p = Ubar Sigma Vbar^T
    U = Qb @ Vb[:, :r]                           # S6  U = Qbar_p Vbar
    V = Q @ Ub[:, :r]                            # S7  V = Q_p Ubar
    U, V = sign_normalize(U, V)
    return RandResult(U=U, S=S[:r].copy(), V=V, R=R, Qbar=Qb, Q=Q)
