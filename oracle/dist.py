"""Row-partitioned LancSVD / RandSVD model on CPU.

ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The multi-GPU path of the library (include/tsvd.h tsvd_create_*_dist) splits
A by rows: rank g owns rows [r0, r1) of A (and of every m-side vector) and the
n-shard [g*ns, min(n, (g+1)*ns)), ns = ceil(n/world), of every n-side vector.
This module runs exactly that decomposition with numpy on each rank and
torch.distributed (gloo) collectives, so the decomposition itself - which sums
are all-reduced, where the reduce-scatter / all-gather sit, which rows of the
Philox blocks each rank draws - is checked against the single-process oracle
on CPU (tests/test_dist_gloo.py).  Per block step of Alg. 2:

  Z_g = A_g^T Qbar_g (full n)  -> reduce-scatter (gloo: all-reduce + slice)
  n-side CGS-CQR2 on the shard, every P^T Y and Y^T Y all-reduced
  Q_i shards -> all-gather -> A_g Q_i (this rank's m rows)
  m-side CGS-CQR2 on the rows, all-reduced projections and Grams
  B_k, its SVD, rho, restart decision: replicated (identical inputs)
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .core import CGS2_TAU, chol, small_svd, trsm_right_lt
from .philox import gaussian_block


class Comm:
    """Sum all-reduce / all-gather of numpy arrays over a torch.distributed group."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def allreduce(self, a):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        self.dist.all_reduce(t)
        return t.numpy()

    def allgather_rows(self, a):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        sizes = [None] * self.world
        self.dist.all_gather_object(sizes, t.shape[0])
        mx = max(sizes)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype)
        pad[:t.shape[0]] = t
        out = [torch.zeros_like(pad) for _ in range(self.world)]
        self.dist.all_gather(out, pad)
        return np.concatenate([o[:s].numpy() for o, s in zip(out, sizes)], axis=0)


class RowShard:
    """This rank's rows of A (CSR or dense) + the n-shard geometry."""

    def __init__(self, comm, m, n, bounds, csr=None, dense=None):
        self.comm, self.m, self.n = comm, m, n
        g = comm.rank
        self.r0, self.r1 = int(bounds[g]), int(bounds[g + 1])
        self.ns = -(-n // comm.world)
        self.n0 = min(n, g * self.ns)
        self.n1 = min(n, self.n0 + self.ns)
        if dense is not None:
            self.A = np.asarray(dense[self.r0:self.r1], dtype=np.float64)
        else:
            rowptr, colidx, vals = csr
            lo, hi = rowptr[self.r0], rowptr[self.r1]
            self.A = sp.csr_matrix((vals[lo:hi], colidx[lo:hi], rowptr[self.r0:self.r1 + 1] - lo),
                                   shape=(self.r1 - self.r0, n))

    def matmul(self, Xshard):
        """A_g X with X given as this rank's n-shard (all-gathered first)."""
        X = self.comm.allgather_rows(Xshard)
        return np.asarray(self.A @ X, dtype=np.float64)

    def rmatmul(self, Xrows):
        """(A^T X)[n-shard] from this rank's rows of X (sum over ranks)."""
        Z = self.comm.allreduce(np.asarray(self.A.T @ Xrows, dtype=np.float64))
        return Z[self.n0:self.n1]


class DrawCtx:
    def __init__(self, seed, row0, q_total):
        self.seed, self.next, self.row0, self.q_total = seed, 1, row0, q_total

    def draw(self, q):
        t = self.next
        self.next += 1
        return gaussian_block(q, 1, self.seed, draw=t, row0=self.row0, q_total=self.q_total)[:, 0]


def cgs2(Y, P, ctx, ar, tau=CGS2_TAU):
    q, w = Y.shape
    s = 0 if P is None else P.shape[1]
    Q = np.zeros((q, w))
    H = np.zeros((s, w))
    R = np.zeros((w, w))
    for j in range(w):
        y = Y[:, j].copy()
        Bm = Q[:, :j] if s == 0 else np.hstack([P, Q[:, :j]])
        c1 = ar(Bm.T @ y)
        y = y - Bm @ c1
        c2 = ar(Bm.T @ y)
        y = y - Bm @ c2
        c = c1 + c2
        nrm = np.sqrt(ar(np.array([y @ y]))[0])
        norig = np.sqrt(ar(np.array([Y[:, j] @ Y[:, j]]))[0])
        if nrm <= tau * norig:
            g = ctx.draw(q)
            for _ in range(2):
                g = g - Bm @ ar(Bm.T @ g)
            Q[:, j] = g / np.sqrt(ar(np.array([g @ g]))[0])
            R[j, j] = 0.0
        else:
            Q[:, j] = y / nrm
            R[j, j] = nrm
        H[:, j] = c[:s]
        R[:j, j] = c[s:]
    return Q, H, R


def cholqr2(Y, ctx, ar):
    L = chol(ar(Y.T @ Y))
    if L is None:
        Q, _, R = cgs2(Y, None, ctx, ar)
        return Q, R
    Q1 = trsm_right_lt(Y, L)
    Lb = chol(ar(Q1.T @ Q1))
    if Lb is None:
        Q, _, R = cgs2(Y, None, ctx, ar)
        return Q, R
    return trsm_right_lt(Q1, Lb), Lb.T @ L.T


def cgs_cqr2(Y, P, ctx, ar):
    if P.shape[1] == 0:
        Q, R = cholqr2(Y, ctx, ar)
        return Q, np.zeros((0, Y.shape[1])), R
    H = ar(P.T @ Y)
    Q0 = Y - P @ H
    L = chol(ar(Q0.T @ Q0))
    if L is None:
        return cgs2(Y, P, ctx, ar)
    Q1 = trsm_right_lt(Q0, L)
    Hb = ar(P.T @ Q1)
    Q2 = Q1 - P @ Hb
    Lb = chol(ar(Q2.T @ Q2))
    if Lb is None:
        return cgs2(Y, P, ctx, ar)
    return trsm_right_lt(Q2, Lb), H + Hb @ L.T, Lb.T @ L.T


def _signs(comm, V):
    Vfull = comm.allgather_rows(V)
    k = np.argmax(np.abs(Vfull), axis=0)
    return np.where(Vfull[k, np.arange(V.shape[1])] < 0, -1.0, 1.0)


def lancsvd_dist(shard: RowShard, r, b, d, tol, maxit, seed):
    """Alg. 2 on a row partition; returns (U rows, S, V n-shard, cycles)."""
    comm = shard.comm
    ar = comm.allreduce
    m_loc = shard.r1 - shard.r0
    n_loc = shard.n1 - shard.n0
    k = d // b
    ctx = DrawCtx(seed, 0, 0)  # one draw counter, rows set per side (as the library)

    def mside():
        ctx.row0, ctx.q_total = shard.r0, shard.m
        return ctx

    def nside():
        ctx.row0, ctx.q_total = shard.n0, shard.n
        return ctx

    G = gaussian_block(m_loc, b, seed, draw=0, row0=shard.r0, q_total=shard.m)
    mctx = mside()
    Qbar, _ = cholqr2(G, mctx, ar)
    for cycle in range(1, maxit + 1):
        Pbar = np.zeros((m_loc, d + b))
        P = np.zeros((n_loc, d))
        B = np.zeros((d, d))
        Pbar[:, :b] = Qbar
        for i in range(k):
            lo, hi = i * b, (i + 1) * b
            Y = shard.rmatmul(Pbar[:, lo:hi])
            nctx = nside()
            if i == 0:
                Q, R = cholqr2(Y, nctx, ar)
            else:
                Q, _, R = cgs_cqr2(Y, P[:, :lo], nctx, ar)
            P[:, lo:hi] = Q
            B[lo:hi, lo:hi] = R.T
            Z = shard.matmul(Q)
            Qb, _, Rb = cgs_cqr2(Z, Pbar[:, :hi], mside(), ar)
            Pbar[:, hi:hi + b] = Qb
            if i < k - 1:
                B[hi:hi + b, lo:hi] = Rb
        Ub, S, Vb = small_svd(B)
        rho = np.linalg.norm(Rb @ Vb[(k - 1) * b:k * b, :], axis=0)
        if np.all(rho[:r] <= tol * S[0]) or cycle == maxit:
            break
        Qbar, _ = cholqr2(Pbar[:, :d] @ Ub[:, :b], mside(), ar)
    V = P @ Vb[:, :r]
    sg = _signs(comm, V)
    return (Pbar[:, :d] @ Ub[:, :r]) * sg, S[:r].copy(), V * sg, cycle


def randsvd_dist(shard: RowShard, r, p, q, b_qr, seed):
    """Alg. 1 on a row partition; returns (U rows, S, V n-shard)."""
    comm = shard.comm
    ar = comm.allreduce
    l = r + p
    n_loc = shard.n1 - shard.n0
    dctx = DrawCtx(seed, 0, 0)

    def mctx_():
        dctx.row0, dctx.q_total = shard.r0, shard.m
        return dctx

    def nctx_():
        dctx.row0, dctx.q_total = shard.n0, shard.n
        return dctx

    def cgs_qr(Y, ctx):
        qq, ll = Y.shape
        Qo = np.zeros((qq, ll))
        Ro = np.zeros((ll, ll))
        for s0 in range(0, ll, b_qr):
            w = min(b_qr, ll - s0)
            if s0 == 0:
                Qj, Rj = cholqr2(Y[:, :w], ctx, ar)
            else:
                Qj, Hj, Rj = cgs_cqr2(Y[:, s0:s0 + w], Qo[:, :s0], ctx, ar)
                Ro[:s0, s0:s0 + w] = Hj
            Qo[:, s0:s0 + w] = Qj
            Ro[s0:s0 + w, s0:s0 + w] = Rj
        return Qo, Ro

    Q = gaussian_block(n_loc, l, seed, draw=0, row0=shard.n0, q_total=shard.n)
    for _ in range(q + 1):
        Qb, _ = cgs_qr(shard.matmul(Q), mctx_())
        Q, R = cgs_qr(shard.rmatmul(Qb), nctx_())
    Ub, S, Vb = small_svd(R)
    V = Q @ Ub[:, :r]
    sg = _signs(comm, V)
    return (Qb @ Vb[:, :r]) * sg, S[:r].copy(), V * sg
