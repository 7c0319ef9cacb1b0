"""Pins for the oracle's building blocks (CPU only, -m "not gpu").

Each test checks the oracle against something other than itself: published
KAT vectors, closed forms, Householder QR from LAPACK (a different routine
than the Cholesky-based ones under test), algebraic identities of the
paper's algorithms, and special cases.
"""
import os

import numpy as np
import pytest

import oracle
from oracle.core import (DrawCtx, chol, trsm_right_lt, cholqr2, cgs_cqr2, bcgs_pip2, cgs2, cgs_qr,
                         small_svd)
from oracle.philox import philox4x32_10, gaussian_from_words, gaussian_block

U = 2.0 ** -53
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([int(x, 16) for x in line.split()])
    return rows


def test_philox_kat():
    rows = _kat()
    assert len(rows) == 3
    for r in rows:
        out = philox4x32_10(tuple(r[0:4]), tuple(r[4:6]))
        assert [int(x) for x in out] == r[6:10]


def test_box_muller_closed_form():
    # a+1 = 2^52  -> u1 = 1/2 ; c = 0 -> u2 = 0  =>  z = sqrt(2 ln 2)
    a = (1 << 52) - 1
    x = a << 11
    w = [np.uint64(x & 0xFFFFFFFF), np.uint64(x >> 32), np.uint64(0), np.uint64(0)]
    z = gaussian_from_words(*w)
    assert z == pytest.approx(np.sqrt(2.0 * np.log(2.0)), rel=1e-15)
    # c = 2^51 -> u2 = 1/4 -> cos(pi/2) ~ 0
    c = (1 << 51) << 11
    w2 = [w[0], w[1], np.uint64(c & 0xFFFFFFFF), np.uint64(c >> 32)]
    assert abs(gaussian_from_words(*w2)) < 1e-15
    # a = 2^53-1 -> u1 = 1 -> z = 0 exactly
    x = ((1 << 53) - 1) << 11
    w3 = [np.uint64(x & 0xFFFFFFFF), np.uint64(x >> 32), np.uint64(123), np.uint64(456)]
    assert gaussian_from_words(*w3) == 0.0


def test_gaussian_statistics_and_partition_independence():
    g = gaussian_block(200_000, 4, seed=0x1234, draw=0)
    assert abs(g.mean()) < 5e-3
    assert abs(g.var() - 1.0) < 1e-2
    kurt = np.mean(g ** 4) / g.var() ** 2
    assert abs(kurt - 3.0) < 0.05
    full = gaussian_block(50, 3, seed=99, draw=2)
    part = gaussian_block(20, 3, seed=99, draw=2, row0=17, q_total=50)
    assert np.array_equal(full[17:37], part)
    assert not np.array_equal(gaussian_block(50, 3, 99, draw=3), full)


def _cond_matrix(q, w, kappa, rng, scale=1.0):
    X, _ = np.linalg.qr(rng.standard_normal((q, w)))
    Y, _ = np.linalg.qr(rng.standard_normal((w, w)))
    s = np.logspace(0, -np.log10(kappa), w) * scale
    return (X * s) @ Y.T


def _householder_posdiag(Y):
    Q, R = np.linalg.qr(Y)
    sg = np.sign(np.diag(R))
    return Q * sg, R * sg[:, None]


@pytest.mark.parametrize("kappa,scale", [(1e2, 1.0), (1e6, 1e3), (1e7, 1e6)])
def test_cholqr2_invariants(kappa, scale):
    rng = np.random.default_rng(1)
    q, w = 400, 12
    Y = _cond_matrix(q, w, kappa, rng, scale)
    Q, R = cholqr2(Y, DrawCtx(0))
    assert np.abs(Q.T @ Q - np.eye(w)).max() <= 10 * w * U
    assert np.linalg.norm(Y - Q @ R) / np.linalg.norm(Y) <= 10 * U * 10
    assert np.allclose(np.tril(R, -1), 0.0)
    assert np.all(np.diag(R) > 0)
    Qh, Rh = _householder_posdiag(Y)
    assert np.abs(Q - Qh).max() <= kappa * 1e-14
    assert np.abs(R - Rh).max() / np.abs(Rh).max() <= kappa * 1e-14


def test_chol_breakdown_detection():
    W = np.array([[1.0, 2.0], [2.0, 1.0]])     # indefinite
    assert chol(W) is None
    W = np.array([[4.0, 2.0], [2.0, 5.0]])
    L = chol(W)
    assert np.array_equal(L, np.array([[2.0, 0.0], [1.0, 2.0]]))
    Y = np.array([[2.0, 1.0], [4.0, 4.0]])
    # Y L^{-T}: solve Q L^T = Y -> row [2,1]: q0 = 1, q1 = (1 - 1*1)/2 = 0
    assert np.allclose(trsm_right_lt(Y, L), [[1.0, 0.0], [2.0, 1.0]])
    assert chol(np.array([[np.nan]])) is None


@pytest.mark.parametrize("kappa", [1.0, 1e4, 1e8])
def test_cgs_cqr2_invariants(kappa):
    rng = np.random.default_rng(2)
    q, s, w = 500, 24, 8
    P, _ = np.linalg.qr(rng.standard_normal((q, s)))
    # Y mostly inside span(P): the remainder is ill conditioned
    Y = P @ rng.standard_normal((s, w)) + _cond_matrix(q, w, kappa, rng, 1e-3)
    Q, H, R = cgs_cqr2(Y, P, DrawCtx(0))
    assert np.abs(P.T @ Q).max() <= 10 * U * 10
    assert np.abs(Q.T @ Q - np.eye(w)).max() <= 10 * w * U
    assert np.linalg.norm(Y - P @ H - Q @ R) / np.linalg.norm(Y) <= 10 * U * 10
    assert np.allclose(np.tril(R, -1), 0.0) and np.all(np.diag(R) > 0)
    # Q = last block of the Householder Q of [P | Y] (positive diagonal)
    Qh, Rh = _householder_posdiag(np.hstack([P, Y]))
    sgn = np.sign(np.diag(Rh)[:s])
    assert np.all(sgn != 0)
    Qlast = Qh[:, s:]
    # P's own block may come out with flipped signs; the last block is fixed
    # by the positive-diagonal convention of R.
    # forward error of a QR factor is O(u * cond): use the condition number
    # of [P | Y] itself
    cond = np.linalg.cond(np.hstack([P, Y]))
    assert np.abs(Q - Qlast).max() <= 1e-14 * cond


@pytest.mark.parametrize("kappa", [1.0, 1e3, 1e6])
def test_bcgs_pip2_invariants(kappa):
    """BCGS-PIP+ (reading R34) pinned by what fixes a block QR:
    Q^T Q = I, P^T Q = 0, Y = P H + Q R with R upper triangular and positive
    diagonal -- so Q equals the last block of the Householder Q of [P | Y]
    and (Q, H, R) equal CGS-CQR2's (the QR with positive diagonal is
    unique) to O(u cond).  A dropped R1 in H = H1 + H2 R1, or R1 R2 for
    R2 R1, breaks Y = P H + Q R here (the second pass is not a no-op in
    floating point, and R1 is far from I)."""
    rng = np.random.default_rng(7)
    q, s, w = 600, 32, 8
    P, _ = np.linalg.qr(rng.standard_normal((q, s)))
    Y = 0.5 * P @ rng.standard_normal((s, w)) + _cond_matrix(q, w, kappa, rng, 3.0)
    Q, H, R = bcgs_pip2(Y, P, DrawCtx(0))
    assert np.abs(P.T @ Q).max() <= 100 * U
    assert np.abs(Q.T @ Q - np.eye(w)).max() <= 10 * w * U
    assert np.linalg.norm(Y - P @ H - Q @ R) / np.linalg.norm(Y) <= 100 * U
    assert np.allclose(np.tril(R, -1), 0.0) and np.all(np.diag(R) > 0)
    cond = np.linalg.cond(np.hstack([P, Y]))
    Qh, Rh = _householder_posdiag(np.hstack([P, Y]))
    assert np.abs(Q - Qh[:, s:]).max() <= 1e-14 * cond
    Qc, Hc, Rc = cgs_cqr2(Y, P, DrawCtx(0))
    assert np.abs(Q - Qc).max() <= 1e-14 * cond
    assert np.abs(R - Rc).max() <= 1e-14 * cond * np.abs(Rc).max()
    assert np.abs(H - Hc).max() <= 1e-14 * cond * np.abs(Hc).max()


def test_bcgs_pip2_breakdown_falls_back_to_cgs2():
    """A column inside span(P) makes W - H^T H singular (the Pythagorean
    Cholesky breaks down): the P:275 fallback gives exactly cgs2's result."""
    rng = np.random.default_rng(4)
    q = 60
    P, _ = np.linalg.qr(rng.standard_normal((q, 5)))
    Y = np.stack([rng.standard_normal(q), P[:, 0] * 3.0, rng.standard_normal(q)], axis=1)
    Q, H, R = bcgs_pip2(Y, P, DrawCtx(11))
    Qd, Hd, Rd = cgs2(Y, P, DrawCtx(11))
    assert np.array_equal(Q, Qd) and np.array_equal(R, Rd) and np.array_equal(H, Hd)
    assert R[1, 1] == 0.0


def test_cgs_cqr2_with_empty_basis_is_cholqr2():
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((100, 5))
    Q1, H, R1 = cgs_cqr2(Y, np.zeros((100, 0)), DrawCtx(0))
    Q2, R2 = cholqr2(Y, DrawCtx(0))
    assert H.shape == (0, 5)
    assert np.array_equal(Q1, Q2) and np.array_equal(R1, R2)


def test_cgs2_fallback_rank_deficient():
    rng = np.random.default_rng(4)
    q = 60
    P, _ = np.linalg.qr(rng.standard_normal((q, 5)))
    a = rng.standard_normal(q)
    Y = np.stack([a, 2.0 * a, P[:, 0] * 3.0, rng.standard_normal(q)], axis=1)
    # Cholesky of the Gram of (Y - P P^T Y) breaks down (col 1 = 2 col 0,
    # col 2 inside span P)
    Q, H, R = cgs_cqr2(Y, P, DrawCtx(11))
    assert np.abs(Q.T @ Q - np.eye(4)).max() < 1e-14
    assert np.abs(P.T @ Q).max() < 1e-14
    assert np.linalg.norm(Y - P @ H - Q @ R) / np.linalg.norm(Y) < 1e-14
    assert R[1, 1] == 0.0 and R[2, 2] == 0.0 and R[0, 0] > 0 and R[3, 3] > 0
    # the direct call gives the same thing
    Qd, Hd, Rd = cgs2(Y, P, DrawCtx(11))
    assert np.array_equal(Q, Qd) and np.array_equal(R, Rd)


def test_cholqr2_breakdown_falls_back():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((50, 2))
    # an exactly zero column makes a Cholesky pivot exactly 0 -> breakdown
    Y = np.hstack([a, np.zeros((50, 1))])
    assert chol(Y.T @ Y) is None
    Q, R = cholqr2(Y, DrawCtx(3))
    assert np.abs(Q.T @ Q - np.eye(3)).max() < 1e-14
    assert np.linalg.norm(Y - Q @ R) / np.linalg.norm(Y) < 1e-14
    assert R[2, 2] == 0.0


@pytest.mark.parametrize("l,bq", [(20, 16), (37, 8), (16, 16), (5, 1)])
def test_cgs_qr_matches_householder(l, bq):
    rng = np.random.default_rng(6)
    Y = _cond_matrix(300, l, 1e5, rng)
    Q, R = cgs_qr(Y, bq, DrawCtx(0))
    assert np.abs(Q.T @ Q - np.eye(l)).max() <= 1e-14
    assert np.linalg.norm(Y - Q @ R) / np.linalg.norm(Y) <= 1e-14
    assert np.allclose(np.tril(R, -1), 0.0)
    Qh, Rh = _householder_posdiag(Y)
    assert np.abs(R - Rh).max() / np.abs(Rh).max() < 1e-9
    assert np.abs(Q - Qh).max() < 1e-9


def test_small_svd_closed_form():
    rng = np.random.default_rng(7)
    d = 30
    s_true = np.sort(rng.random(d) * 5)[::-1]
    Pm = np.eye(d)[rng.permutation(d)]
    Qm = np.eye(d)[rng.permutation(d)]
    signs = rng.choice([-1.0, 1.0], size=d)
    B = Pm @ np.diag(s_true * signs) @ Qm.T
    Ub, S, Vb = small_svd(B)
    assert np.abs(S - s_true).max() <= 4 * U * s_true[0]
    assert np.abs(Ub @ np.diag(S) @ Vb.T - B).max() <= 4 * U * s_true[0]
    # lower block bidiagonal random B: invariants
    B = np.tril(rng.standard_normal((d, d))) - np.tril(rng.standard_normal((d, d)), -8)
    Ub, S, Vb = small_svd(B)
    assert np.all(np.diff(S) <= 0)
    assert np.abs(Ub @ np.diag(S) @ Vb.T - B).max() < 1e-13 * S[0]
    assert np.abs(Ub.T @ Ub - np.eye(d)).max() < 1e-13


def test_sign_normalize():
    U = np.array([[1.0, 2.0], [3.0, 4.0]])
    V = np.array([[0.1, -0.9], [-0.5, 0.2]])
    Un, Vn = oracle.sign_normalize(U, V)
    assert np.array_equal(Vn[:, 0], [-0.1, 0.5]) and np.array_equal(Un[:, 0], [-1.0, -3.0])
    assert np.array_equal(Vn[:, 1], [0.9, -0.2]) and np.array_equal(Un[:, 1], [-2.0, -4.0])
