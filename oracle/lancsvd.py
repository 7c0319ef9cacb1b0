"""LancSVD: block Golub-Kahan-Lanczos truncated SVD with full
reorthogonalisation and basic restart.  Alg. 2.

ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation: the paper's Krylov dimension "r" is d here (k = d/b
block steps per cycle); the paper's restart count "p" is maxit (with an early
exit on tol, reading R12); r is the number of wanted triplets.

Readings applied: both sides are orthogonalised (R15);
B_k[i,i] = L_i = R^T of the S3 factorisation, B_k[i+1,i] = Rbar_i (Eq. 8,
R17, R1); Qbar_{k+1} is kept to supply Rbar_k (R18); the restart block is the
first b left Ritz vectors (R19) re-orthonormalised with CholQR2 (R11);
V_r = P_k Vbar (Eq. 12, R2); convergence rho_i = ||Rbar_k Vbar[last b, i]||
<= tol * sigma_1 (from Eq. 10, R12).

keep = l > 0 selects the THICK restart (the paper's own
future work, after Baglama-Reichel, ref. [2] P:509) instead
of Alg. 2 S7.  It is not in the paper's listing, so it is written from the
Lanczos relations of Eq. 7 (reading R1) that the listing maintains:
  A P_k = Pbar_k B_k + Qbar_{k+1} Rbar_k E_k^T,   A^T Pbar_k = P_k B_k^T.
With B_k = Ubar Sigma Vbar^T, the l largest Ritz vectors Pbar' = Pbar_k
Ubar[:, :l], P' = P_k Vbar[:, :l] satisfy
  A P' = Pbar' Sigma_l + Qbar_{k+1} S,  S = Rbar_k Vbar[last b rows, :l],
  A^T Pbar' = P' Sigma_l,
so the next cycle starts from Pbar = [Pbar' | Qbar_{k+1}], P = [P'], and
continues the block recurrence (S2-S5, full reorthogonalisation) for
(d - l)/b block steps.  Its projected matrix B' = Pbar^T A P is
  [ Sigma_l   0    0  ... ]
  [ S         L_1  0  ... ]      (lower "arrow" + block bidiagonal)
  [ 0         Rb_1 L_2 ...]
and rho_i, the outputs and the convergence test are unchanged.  l must be a
multiple of b (d - l too); l >= r is required.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import DrawCtx, bcgs_pip2, cholqr2, cgs_cqr2, small_svd, sign_normalize
from .philox import gaussian_block


@dataclass
class LancResult:
    U: np.ndarray
    S: np.ndarray
    V: np.ndarray
    rho: np.ndarray
    cycles: int
    nconv: int
    converged: bool
    debug: dict = field(default_factory=dict)


def lancsvd(op, r: int, b: int, d: int, tol: float, maxit: int, seed: int,
            start=None, debug: bool = False, keep: int = 0,
            ortho: str = "cgs_cqr2") -> LancResult:
    """ortho: the block orthogonalisation of S3b / S5 -- "cgs_cqr2" (the
    paper's Alg. 5) or "bcgs_pip2" (SURVEY 8(f) N2 ablation, core.bcgs_pip2)."""
    m, n = op.m, op.n
    orth = {"cgs_cqr2": cgs_cqr2, "bcgs_pip2": bcgs_pip2}[ortho]
    assert m >= n and 1 <= r <= d <= n and d % b == 0 and maxit >= 1
    assert keep == 0 or (keep % b == 0 and r <= keep < d)
    ctx = DrawCtx(seed)
    G = gaussian_block(m, b, seed, draw=0) if start is None else np.array(start, dtype=np.float64)
    Qbar, _ = cholqr2(G, ctx)                                   # S1
    thick = None
    for cycle in range(1, maxit + 1):                            # j = 1..p
        Pbar = np.zeros((m, d + b))
        P = np.zeros((n, d))
        B = np.zeros((d, d))
        s0 = 0
        if thick is None:
            Pbar[:, 0:b] = Qbar
        else:                                                    # N1: thick restart
            s0 = keep
            Pbar_o, P_o, Ub_o, S_o, Vb_o, Rb_o = thick
            Pbar[:, :s0] = Pbar_o[:, :d] @ Ub_o[:, :s0]
            P[:, :s0] = P_o @ Vb_o[:, :s0]
            Pbar[:, s0:s0 + b] = Pbar_o[:, d:d + b]              # Qbar_{k+1}
            B[:s0, :s0] = np.diag(S_o[:s0])
            B[s0:s0 + b, :s0] = Rb_o @ Vb_o[d - b:d, :s0]        # S
        k = (d - s0) // b
        Rb = None
        for i in range(k):                                       # i = 1..k
            lo, hi = s0 + i * b, s0 + (i + 1) * b
            Y = op.rmatmul(Pbar[:, lo:hi])                       # S2
            if lo == 0:
                Q, R = cholqr2(Y, ctx)                           # S3a
            else:
                Q, _, R = orth(Y, P[:, :lo], ctx)                # S3b
            P[:, lo:hi] = Q
            B[lo:hi, lo:hi] = R.T                                # L_i
            Z = op.matmul(Q)                                     # S4
            Qb, _, Rb = orth(Z, Pbar[:, :hi], ctx)               # S5
            Pbar[:, hi:hi + b] = Qb
            if i < k - 1:
                B[hi:hi + b, lo:hi] = Rb                         # Rbar_i
        Ub, S, Vb = small_svd(B)                                 # SVD(B_k)
        rho = np.linalg.norm(Rb @ Vb[d - b:d, :], axis=0)
        ok = rho[:r] <= tol * S[0]
        converged = bool(np.all(ok))
        if converged or cycle == maxit:
            break
        if keep:
            thick = (Pbar, P, Ub, S, Vb, Rb)
        else:
            Qbar, _ = cholqr2(Pbar[:, :d] @ Ub[:, :b], ctx)      # S7 (+R11)
    U = Pbar[:, :d] @ Ub[:, :r]                                  # S9
    V = P @ Vb[:, :r]                                            # S8 (Eq. 12)
    U, V = sign_normalize(U, V)
    dbg = {}
    if debug:
        dbg = dict(B=B, P=P, Pbar=Pbar[:, :d], Qnext=Pbar[:, d:d + b], Rbar=Rb,
                   Ub=Ub, Vb=Vb, S_all=S)
    return LancResult(U=U, S=S[:r].copy(), V=V, rho=rho[:r].copy(), cycles=cycle,
                      nconv=int(np.sum(ok)), converged=converged, debug=dbg)


def default_krylov_dim(r: int, b: int, n: int) -> int:
    """d when none is given: min(n, max(4 r, 2 b), 1536) rounded down to a
    multiple of b (include/tsvd.h, tsvd_set_krylov_dim; 1536 = the largest
    B_k the library's device SVD takes)."""
    d = min(max(4 * r, 2 * b), n, 1536)
    return d - d % b


def lancsvd_threshold(op, tau: float, b: int, tol: float, maxit: int, r_max: int, seed: int,
                      d: int | None = None):
    """the rank set by the threshold of Eq. 3,
    ||A - U_r S_r V_r^T||_2 = sigma_{r+1} <= tau * sigma_1.  Reading R33:
    LancSVD is run for r + 1 wanted triplets (r = b first, then doubled up to
    r_max, each run from the same fresh start); the answer is the smallest r
    with sigma_{r+1} <= tau * sigma_1 whose triplets 1..r+1 converged
    (rho <= tol * sigma_1).  Returns (LancResult trimmed to r, r, found)."""
    r_max = min(r_max, op.n - 1)
    req = min(b, r_max)
    while True:
        want = req + 1
        dd = d if d else default_krylov_dim(want, b, op.n)
        res = lancsvd(op, want, b, dd, tol, maxit, seed)
        conv = res.rho <= tol * res.S[0]
        found = None
        for r in range(1, want):
            if not (conv[r - 1] and conv[r]):
                break
            if res.S[r] <= tau * res.S[0]:
                found = r
                break
        if found is not None or req >= r_max:
            r = found if found is not None else req
            out = LancResult(U=res.U[:, :r].copy(), S=res.S[:r].copy(), V=res.V[:, :r].copy(),
                             rho=res.rho[:r].copy(), cycles=res.cycles,
                             nconv=int(np.sum(conv[:r])), converged=found is not None)
            return out, r, found is not None
        req = min(2 * req, r_max)
