"""Building blocks of RandSVD / LancSVD, written from the paper.

ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  Operator        products A.X and A^T.X (Alg. 1 S1/S3, Alg. 2 S2/S4)
  chol            Cholesky with the breakdown test of P:275
  trsm_right_lt   Q = Y L^{-T}  (Alg. 4 S3/S6, Alg. 5 S5/S10)
  cholqr2         Alg. 4, S5 typo and S7 order corrected
  cgs_cqr2        Alg. 5, S11 order and S12 corrected
  cgs2            P:275 fallback: column-wise CGS with reorthogonalisation
  cgs_qr          Alg. 3, ragged last panel allowed
  small_svd       Alg. 1 S5 / Alg. 2 SVD(B_k): LAPACK GESVD (Table 1)
  sign_normalize  DESIGN.md reading R28
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .philox import gaussian_block

CGS2_TAU = 1e-13  # DESIGN.md reading R16 (dependent-column threshold)


class Operator:
    """The m x n matrix A of Sec. 2, m >= n, dense or CSR."""

    def __init__(self, dense=None, csr=None, shape=None):
        if dense is not None:
            self.A = np.asarray(dense, dtype=np.float64)
            self.m, self.n = self.A.shape
            self.kind = "dense"
        else:
            rowptr, colidx, vals = csr
            self.m, self.n = shape
            self.A = sp.csr_matrix((np.asarray(vals, np.float64),
                                    np.asarray(colidx, np.int64),
                                    np.asarray(rowptr, np.int64)),
                                   shape=shape)
            self.kind = "csr"

    def matmul(self, X):
        """A . X  (Alg. 1 S1, Alg. 2 S4)."""
        return np.asarray(self.A @ X, dtype=np.float64)

    def rmatmul(self, X):
        """A^T . X  (Alg. 1 S3, Alg. 2 S2)."""
        return np.asarray(self.A.T @ X, dtype=np.float64)

    def todense(self):
        return self.A if self.kind == "dense" else self.A.toarray()


class DrawCtx:
    """Philox draw bookkeeping: draw 0 is the start block; each
    breakdown replacement column takes the next draw id (reading R16)."""

    def __init__(self, seed: int):
        self.seed = seed
        self.next = 1

    def draw(self, q: int):
        t = self.next
        self.next += 1
        return gaussian_block(q, 1, self.seed, draw=t)[:, 0]


def chol(W):
    """W = L L^T (Alg. 4 S2/S5).  Breakdown iff a pivot is <= 0 or
    non-finite: returns None."""
    if not np.all(np.isfinite(W)):
        return None
    try:
        L = np.linalg.cholesky(W)
    except np.linalg.LinAlgError:
        return None
    if not np.all(np.isfinite(L)) or np.any(np.diag(L) <= 0.0):
        return None
    return L


def trsm_right_lt(Y, L):
    """Q = Y L^{-T}, i.e. solve Q L^T = Y (Alg. 4 S3)."""
    return sla.solve_triangular(L, Y.T, lower=True).T


def cgs2(Y, P, ctx: DrawCtx, tau: float = CGS2_TAU):
    """Fallback of P:275: classical Gram-Schmidt with reorthogonalisation,
    one column at a time, against [P, Q_<j].  A column whose remainder is
    <= tau*||y_j|| is replaced by a fresh Philox column orthogonalised the
    same way, with R[j,j] = 0 (reading R16).  Returns (Q, H, R) with
    Y = P H + Q R."""
    q, w = Y.shape
    s = 0 if P is None else P.shape[1]
    Q = np.zeros((q, w))
    H = np.zeros((s, w))
    R = np.zeros((w, w))
    for j in range(w):
        y = Y[:, j].copy()
        Bm = Q[:, :j] if s == 0 else np.hstack([P, Q[:, :j]])
        c1 = Bm.T @ y
        y = y - Bm @ c1
        c2 = Bm.T @ y
        y = y - Bm @ c2
        c = c1 + c2
        nrm = np.linalg.norm(y)
        if nrm <= tau * np.linalg.norm(Y[:, j]):
            g = ctx.draw(q)
            for _ in range(2):
                g = g - Bm @ (Bm.T @ g)
            Q[:, j] = g / np.linalg.norm(g)
            R[j, j] = 0.0
        else:
            Q[:, j] = y / nrm
            R[j, j] = nrm
        H[:, j] = c[:s]
        R[:j, j] = c[s:]
    return Q, H, R


def cholqr2(Y, ctx: DrawCtx):
    """Alg. 4 CholeskyQR2.  Returns (Q, R), Y = Q R.
    S5 factorises W-bar (typo in print, reading R3); S7 is R = Lbar^T L^T
    (printed L^T Lbar^T is wrong unless Lbar = I; reading R4)."""
    W = Y.T @ Y                      # S1
    L = chol(W)                      # S2
    if L is None:
        Q, _, R = cgs2(Y, None, ctx)
        return Q, R
    Q1 = trsm_right_lt(Y, L)         # S3
    Wb = Q1.T @ Q1                   # S4
    Lb = chol(Wb)                    # S5
    if Lb is None:
        Q, _, R = cgs2(Y, None, ctx)
        return Q, R
    Q = trsm_right_lt(Q1, Lb)        # S6
    R = Lb.T @ L.T                   # S7 (corrected)
    return Q, R


def cgs_cqr2(Y, P, ctx: DrawCtx):
    """Alg. 5 CGS-CQR2.  Returns (Q, H, R) with
    Y = P H + Q R.  S11: R = Lbar^T L^T; S12: H = H + Hbar L^T (readings
    R4, R5)."""
    if P is None or P.shape[1] == 0:
        Q, R = cholqr2(Y, ctx)
        return Q, np.zeros((0, Y.shape[1])), R
    H = P.T @ Y                      # S1
    Q0 = Y - P @ H                   # S2
    W = Q0.T @ Q0                    # S3
    L = chol(W)                      # S4
    if L is None:
        return cgs2(Y, P, ctx)
    Q1 = trsm_right_lt(Q0, L)        # S5
    Hb = P.T @ Q1                    # S6
    Q2 = Q1 - P @ Hb                 # S7
    Wb = Q2.T @ Q2                   # S8
    Lb = chol(Wb)                    # S9
    if Lb is None:
        return cgs2(Y, P, ctx)
    Q = trsm_right_lt(Q2, Lb)        # S10
    R = Lb.T @ L.T                   # S11 (corrected)
    H = H + Hb @ L.T                 # S12 (corrected)
    return Q, H, R


def bcgs_pip2(Y, P, ctx: DrawCtx):
    """BCGS-PIP+ (reading R34): block classical Gram-Schmidt
    with the Pythagorean inner product, run twice (reorthogonalisation).
    NOT in the paper: the communication-reducing alternative to Alg. 5
    (CGS-CQR2) whose every pass needs ONE reduction, [P Y]^T Y, instead of
    two (P^T Y, then the Gram of the projected block), and no separate pass
    for the TRSM.  Written from its definition (block Gram-Schmidt with the
    Pythagorean Cholesky; Barlow 2019, Carson et al. 2022):
      pass(Y):  H = P^T Y,  W = Y^T Y          (one reduction)
                L = chol(W - H^T H)            (Pythagorean: = Y'^T Y', Y' = Y - P H)
                Q = (Y - P H) L^{-T},  R = L^T
      Q1, H1, R1 = pass(Y);  Q, H2, R2 = pass(Q1)
      H = H1 + H2 R1,  R = R2 R1               (Y = P H + Q R)
    Breakdown (a pivot <= 0 or non-finite in either pass) -> the same CGS2
    fallback as Alg. 5 (reading R16).  Returns (Q, H, R)."""
    if P is None or P.shape[1] == 0:
        Q, R = cholqr2(Y, ctx)
        return Q, np.zeros((0, Y.shape[1])), R

    def one_pass(Z):
        H = P.T @ Z
        W = Z.T @ Z
        L = chol(W - H.T @ H)
        if L is None:
            return None
        return trsm_right_lt(Z - P @ H, L), H, L.T

    p1 = one_pass(Y)
    if p1 is None:
        return cgs2(Y, P, ctx)
    Q1, H1, R1 = p1
    p2 = one_pass(Q1)
    if p2 is None:
        return cgs2(Y, P, ctx)
    Q, H2, R2 = p2
    return Q, H1 + H2 @ R1, R2 @ R1


def cgs_qr(Y, bq: int, ctx: DrawCtx):
    """Alg. 3 CGS-QR with panels of bq columns; the last panel
    may be narrower (reading R8).  Returns (Q, R), R block upper triangular
    with column blocks [H_j; R_j]."""
    q, l = Y.shape
    Q = np.zeros((q, l))
    R = np.zeros((l, l))
    for s in range(0, l, bq):
        w = min(bq, l - s)
        if s == 0:
            Qj, Rj = cholqr2(Y[:, 0:w], ctx)               # S1
        else:
            Qj, Hj, Rj = cgs_cqr2(Y[:, s:s + w], Q[:, :s], ctx)   # S2
            R[:s, s:s + w] = Hj
        Q[:, s:s + w] = Qj
        R[s:s + w, s:s + w] = Rj
    return Q, R


def small_svd(B):
    """SVD of the small projected matrix (Alg. 1 S5, Alg. 2 after the i-loop),
    LAPACK GESVD on the CPU exactly as in Table 1.  Returns
    (Ubar, sigma descending, Vbar) with B = Ubar diag(sigma) Vbar^T."""
    U, s, Vt = sla.svd(B, full_matrices=False, lapack_driver="gesvd")
    return U, s, Vt.T


def sign_normalize(U, V):
    """Flip (u_i, v_i) so the largest-|.| entry of v_i is positive, lowest
    index on ties (reading R28).  Returns copies."""
    U = U.copy()
    V = V.copy()
    for i in range(V.shape[1]):
        k = int(np.argmax(np.abs(V[:, i])))
        if V[k, i] < 0:
            U[:, i] = -U[:, i]
            V[:, i] = -V[:, i]
    return U, V
