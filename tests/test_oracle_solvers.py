"""Pins for the oracle's solvers and the input generators (CPU, -m "not gpu").

Closed forms (prescribed spectra of Eq. 15/16 and of the G2 generator),
the Lanczos relations of Eq. 7-12 (corrected, readings R1/R2), RandSVD's
Eq. 4, special cases (d = n, l = n, b = 1, diagonal A, rank-deficient A) and
Eckart-Young (Eq. 3).
"""
import os

import numpy as np
import pytest

import oracle
from tsvd_inputs import (spectrum_eq16, dense_prescribed, powerlaw_csr,
                         blockdiag_csr, SEEDS)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _c1():
    s = spectrum_eq16(100)
    A = dense_prescribed(200, 100, s, SEEDS["C1"])
    return oracle.Operator(dense=A), s


def test_eq16_spectrum_matches_golden():
    exps = []
    with open(os.path.join(GOLD, "eq16_spectrum_n100.txt")) as f:
        for line in f:
            if line.startswith("#"):
                continue
            exps.append(float(line.split()[1]))
    s = spectrum_eq16(100)
    assert np.allclose(np.log10(s), exps, atol=1e-12)
    assert s[0] == 10.0 and s[10] == pytest.approx(0.01, rel=1e-14)


@pytest.mark.parametrize("refl", [None, 4])
def test_dense_prescribed_has_prescribed_spectrum(refl):
    s = spectrum_eq16(60)
    A = dense_prescribed(150, 60, s, seed=5, n_reflectors=refl)
    sv = np.linalg.svd(A, compute_uv=False)
    assert np.abs(sv - s).max() <= 1e-14 * s[0]


def test_powerlaw_csr_shape_and_skew():
    m, n, nnz = 20000, 20000, 200000
    rowptr, col, val = powerlaw_csr(m, n, nnz, 2.5, seed=3)
    assert rowptr[0] == 0 and rowptr[-1] == len(col) == len(val)
    assert 0.95 * nnz <= len(col) <= nnz
    L = np.diff(rowptr)
    assert L.max() > 20 * L.mean()            # power-law rows
    for i in np.random.default_rng(0).integers(0, m, 200):   # canonical
        c = col[rowptr[i]:rowptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    cc = np.bincount(col, minlength=n)
    assert cc.max() > 20 * cc.mean()          # power-law columns too


def test_blockdiag_csr_spectrum_closed_form():
    top = np.linspace(100.0, 50.0, 20)
    rowptr, col, val, sig = blockdiag_csr(600, 400, 6.0, 2.5, seed=9, top_sigma=top)
    op = oracle.Operator(csr=(rowptr, col, val), shape=(600, 400))
    sv = np.linalg.svd(op.todense(), compute_uv=False)
    assert np.abs(sv - sig[:400]).max() <= 1e-13 * sig[0]
    assert np.allclose(sig[:20], top)


@pytest.mark.parametrize("ortho", ["cgs_cqr2", "bcgs_pip2"])
def test_lancsvd_c1_closed_form(ortho):
    op, s = _c1()
    res = oracle.lancsvd(op, r=10, b=4, d=28, tol=1e-12, maxit=8, seed=SEEDS["C1"], debug=True,
                         ortho=ortho)
    assert res.converged
    assert np.abs(res.S - s[:10]).max() / s[0] <= 1e-10
    e, _ = oracle.residuals(op, res.U, res.S, res.V)
    assert e.max() <= 1e-8
    assert np.abs(res.U.T @ res.U - np.eye(10)).max() <= 1e-12
    assert np.abs(res.V.T @ res.V - np.eye(10)).max() <= 1e-12
    ey = oracle.eckart_young_2norm(op, res.U, res.S, res.V)
    assert ey == pytest.approx(s[10], rel=1e-6)


def _lanczos_relations(op, res, b):
    dbg = res.debug
    A = op.todense()
    P, Pb, B, Qn, Rb = dbg["P"], dbg["Pbar"], dbg["B"], dbg["Qnext"], dbg["Rbar"]
    d = B.shape[0]
    nA = np.linalg.norm(A, 2)
    E = np.zeros((d, b))
    E[d - b:, :] = np.eye(b)
    # Eq. 7 second line / Eq. 10 (reading R1): A P = Pbar B + Qbar_{k+1} Rbar E^T
    r1 = np.linalg.norm(A @ P - Pb @ B - Qn @ Rb @ E.T, 2) / nA
    # Pbar^T A P = B (B lower block bidiagonal, Eq. 8)
    r2 = np.linalg.norm(Pb.T @ A @ P - B, 2) / nA
    o1 = np.abs(P.T @ P - np.eye(d)).max()
    o2 = np.abs(Pb.T @ Pb - np.eye(d)).max()
    return r1, r2, o1, o2


@pytest.mark.parametrize("ortho", ["cgs_cqr2", "bcgs_pip2"])
@pytest.mark.parametrize("b,d", [(4, 28), (1, 12), (3, 24), (5, 100)])
def test_lancsvd_relations(b, d, ortho):
    op, s = _c1()
    res = oracle.lancsvd(op, r=min(10, d), b=b, d=d, tol=1e-30, maxit=1,
                         seed=SEEDS["C1"] + b, debug=True, ortho=ortho)
    r1, r2, o1, o2 = _lanczos_relations(op, res, b)
    assert r1 <= 1e-13 and r2 <= 1e-12 and o1 <= 1e-13 and o2 <= 1e-13
    B = res.debug["B"]
    # block structure of Eq. 8: zero above the diagonal blocks' upper
    # triangle and below the first sub-diagonal block
    k = d // b
    for i in range(k):
        for j in range(k):
            blk = B[i * b:(i + 1) * b, j * b:(j + 1) * b]
            if j > i or i > j + 1:
                assert np.all(blk == 0.0)
            elif i == j:
                assert np.all(np.triu(blk, 1) == 0.0)     # L_i lower
            else:
                assert np.all(np.tril(blk, -1) == 0.0)    # Rbar_i upper
    # rho (from Eq. 10) equals the explicit residual
    e, _ = oracle.residuals(op, res.U, res.S, res.V)
    assert np.abs(res.rho - e * res.S[0]).max() <= 1e-13 * s[0]


def test_lancsvd_full_dimension_is_exact_svd():
    op, s = _c1()
    res = oracle.lancsvd(op, r=100, b=4, d=100, tol=1e-30, maxit=1, seed=1)
    sv = np.linalg.svd(op.A, compute_uv=False)   # LAPACK gesdd (other driver)
    assert np.abs(res.S - sv).max() <= 1e-14 * s[0]


def test_lancsvd_b1_is_golub_kahan():
    op, s = _c1()
    res = oracle.lancsvd(op, r=5, b=1, d=20, tol=1e-30, maxit=1, seed=2, debug=True)
    B = res.debug["B"]
    assert np.all(np.tril(B, -2) == 0.0) and np.all(np.triu(B, 1) == 0.0)
    assert np.abs(res.S - s[:5]).max() <= 1e-10 * s[0]


def test_lancsvd_diagonal_csr():
    n = 300
    rng = np.random.default_rng(3)
    dvals = rng.random(n) + 0.5
    dvals[:8] = [50, 40, 30, 20, 15, 12, 10, 9]
    rowptr = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    op = oracle.Operator(csr=(rowptr, col, dvals), shape=(n, n))
    res = oracle.lancsvd(op, r=6, b=4, d=40, tol=1e-10, maxit=10, seed=4)
    assert res.converged
    assert np.abs(res.S - np.sort(dvals)[::-1][:6]).max() <= 1e-10 * 50
    # V is a set of unit vectors +-e_i up to rounding
    for i in range(6):
        j = int(np.argmax(np.abs(res.V[:, i])))
        assert abs(res.V[j, i] - 1.0) < 1e-10


def test_lancsvd_restarts_converge():
    # slowly decaying spectrum: one cycle of d=16 is not enough; restarts help
    n = 120
    s = 10.0 * 0.93 ** np.arange(n)
    A = dense_prescribed(240, n, s, seed=8)
    op = oracle.Operator(dense=A)
    res = oracle.lancsvd(op, r=4, b=4, d=16, tol=1e-10, maxit=60, seed=5)
    assert res.cycles > 1
    assert res.converged
    assert np.abs(res.S - s[:4]).max() <= 1e-10 * s[0]
    e, _ = oracle.residuals(op, res.U, res.S, res.V)
    assert e.max() <= 1e-8
    assert np.abs(res.U.T @ res.U - np.eye(4)).max() <= 1e-12


def test_lancsvd_rank_deficient_breakdown():
    rng = np.random.default_rng(6)
    m, n, k = 80, 40, 5
    X, _ = np.linalg.qr(rng.standard_normal((m, k)))
    Y, _ = np.linalg.qr(rng.standard_normal((n, k)))
    sv = np.array([5.0, 4.0, 3.0, 2.0, 1.0])
    A = (X * sv) @ Y.T
    op = oracle.Operator(dense=A)
    res = oracle.lancsvd(op, r=5, b=2, d=12, tol=1e-10, maxit=3, seed=7, debug=True)
    assert np.abs(res.S - sv).max() <= 1e-12 * 5
    r1, r2, o1, o2 = _lanczos_relations(op, res, 2)
    assert o1 <= 1e-13 and o2 <= 1e-13 and r2 <= 1e-12


def test_randsvd_full_width_is_exact():
    op, s = _c1()
    for q in (0, 1):
        res = oracle.randsvd(op, r=10, p=90, q=q, b_qr=16, seed=3)
        sv = np.linalg.svd(op.A, compute_uv=False)
        assert np.abs(res.S - sv[:10]).max() <= 1e-13 * s[0]


def test_randsvd_c1_and_eq4():
    op, s = _c1()
    res = oracle.randsvd(op, r=10, p=10, q=1, b_qr=16, seed=SEEDS["C1"])
    assert np.abs(res.S - s[:10]).max() / s[0] <= 1e-10
    e, _ = oracle.residuals(op, res.U, res.S, res.V)
    assert e.max() <= 1e-8
    # Eq. 4: A^T Qbar_p = Q_p R_p
    lhs = op.rmatmul(res.Qbar)
    assert np.linalg.norm(lhs - res.Q @ res.R) / np.linalg.norm(lhs) <= 1e-14
    assert np.abs(res.U.T @ res.U - np.eye(10)).max() <= 1e-12
    # q = 0 (direct method) is less accurate than q = 1 here
    r0 = oracle.randsvd(op, r=10, p=10, q=0, b_qr=16, seed=SEEDS["C1"])
    e0, _ = oracle.residuals(op, r0.U, r0.S, r0.V)
    assert e0.max() > e.max()


def test_spmm_oracle_matches_dense_and_diagonal():
    rowptr, col, val = powerlaw_csr(300, 200, 3000, 2.5, seed=1)
    op = oracle.Operator(csr=(rowptr, col, val), shape=(300, 200))
    X = np.random.default_rng(2).standard_normal((200, 7))
    Xt = np.random.default_rng(3).standard_normal((300, 7))
    D = np.zeros((300, 200))
    for i in range(300):
        for kk in range(rowptr[i], rowptr[i + 1]):
            D[i, col[kk]] += val[kk]
    assert np.abs(op.matmul(X) - D @ X).max() <= 1e-13 * np.abs(D).sum(1).max() * np.abs(X).max()
    assert np.abs(op.rmatmul(Xt) - D.T @ Xt).max() <= 1e-12
    # diagonal: products are exact
    dv = np.random.default_rng(4).standard_normal(50)
    opd = oracle.Operator(csr=(np.arange(51), np.arange(50), dv), shape=(50, 50))
    Xd = np.random.default_rng(5).standard_normal((50, 3))
    assert np.array_equal(opd.matmul(Xd), dv[:, None] * Xd)


# ---- N1 thick restart (oracle/lancsvd.py header) -------------
def _slow_decay(n=120, m=240, seed=8):
    s = 10.0 * 0.93 ** np.arange(n)
    return oracle.Operator(dense=dense_prescribed(m, n, s, seed=seed)), s


@pytest.mark.parametrize("b,d,keep", [(4, 20, 8), (2, 16, 6), (3, 24, 12)])
def test_thick_restart_relations(b, d, keep):
    """After >= 1 thick restart the Lanczos relation A P = Pbar B + Qbar R E^T
    and Pbar^T A P = B (arrow + block bidiagonal) still hold, the bases stay
    orthonormal, and rho equals the explicit residual."""
    op, s = _slow_decay()
    res = oracle.lancsvd(op, r=4, b=b, d=d, tol=1e-30, maxit=3, seed=11, debug=True, keep=keep)
    assert res.cycles == 3
    r1, r2, o1, o2 = _lanczos_relations(op, res, b)
    assert r1 <= 1e-13 and r2 <= 1e-12 and o1 <= 1e-13 and o2 <= 1e-13
    B = res.debug["B"]
    # structure: diagonal Sigma_l block, S row block below it, zeros elsewhere
    assert np.all(B[:keep, :keep] == np.diag(np.diag(B[:keep, :keep])))
    assert np.all(B[:keep, keep:] == 0.0)
    assert np.all(B[keep + b:, :keep] == 0.0)
    assert np.all(np.diff(np.diag(B[:keep, :keep])) <= 0)   # the kept Ritz values, sorted
    e, _ = oracle.residuals(op, res.U, res.S, res.V)
    assert np.abs(res.rho - e * res.S[0]).max() <= 1e-13 * s[0]


def test_thick_restart_first_cycle_equals_paper_restart():
    op, _ = _slow_decay()
    a = oracle.lancsvd(op, r=4, b=4, d=20, tol=1e-30, maxit=1, seed=3, keep=8)
    b_ = oracle.lancsvd(op, r=4, b=4, d=20, tol=1e-30, maxit=1, seed=3)
    assert np.array_equal(a.S, b_.S) and np.array_equal(a.U, b_.U)


def test_thick_restart_converges_where_paper_restart_stalls():
    """C1 with d = 20 < 28: the paper's restart keeps only b = 4 Ritz vectors
    and stalls (SURVEY 7.3 [calib]); keeping l = 12 >= r converges to the
    prescribed Eq. 16 spectrum (closed form) in a few cycles."""
    op, s = _c1()
    res = oracle.lancsvd(op, r=10, b=4, d=20, tol=1e-12, maxit=10, seed=SEEDS["C1"], keep=12)
    assert res.converged and res.cycles <= 4
    assert np.abs(res.S - s[:10]).max() / s[0] <= 1e-10
    e, _ = oracle.residuals(op, res.U, res.S, res.V)
    assert e.max() <= 1e-8
    assert np.abs(res.U.T @ res.U - np.eye(10)).max() <= 1e-12
    assert np.abs(res.V.T @ res.V - np.eye(10)).max() <= 1e-12
    ey = oracle.eckart_young_2norm(op, res.U, res.S, res.V)
    assert ey == pytest.approx(s[10], rel=1e-6)


def test_thick_restart_slow_decay_closed_form():
    op, s = _slow_decay()
    res = oracle.lancsvd(op, r=4, b=4, d=16, tol=1e-10, maxit=60, seed=5, keep=8)
    paper = oracle.lancsvd(op, r=4, b=4, d=16, tol=1e-10, maxit=60, seed=5)
    assert res.converged and res.cycles < paper.cycles
    assert np.abs(res.S - s[:4]).max() <= 1e-10 * s[0]


# ---- N4: rank by threshold (Eq. 3), reading R33 ---------------------------
def test_threshold_rank_closed_form():
    """C1 (Eq. 16 set reading, n = 100): sigma_i = 10^(1 - 0.3 (i - 1)), so
    with tau = 1.5e-3 the smallest r with sigma_{r+1} <= tau sigma_1 = 0.015
    is r = 10 (sigma_10 = 0.01995 > 0.015 >= sigma_11 = 0.01): found after
    the requests r = 4, 8, 16; sigma and Eckart-Young (Eq. 3) pinned by the
    prescribed spectrum."""
    op, s = _c1()
    i = np.arange(1, 12)
    assert np.allclose(s[:11], 10.0 ** (1 - 0.3 * (i - 1)), rtol=1e-14)
    res, r, found = oracle.lancsvd_threshold(op, tau=1.5e-3, b=4, tol=1e-12, maxit=8,
                                             r_max=40, seed=SEEDS["C1"])
    assert found and r == 10
    assert np.abs(res.S - s[:10]).max() / s[0] <= 1e-10
    ey = oracle.eckart_young_2norm(op, res.U, res.S, res.V)
    assert ey == pytest.approx(s[10], rel=1e-6)
    assert ey <= 1.5e-3 * s[0]
    # one step coarser threshold: sigma_10 <= 0.02 -> r = 9
    _, r2, found2 = oracle.lancsvd_threshold(op, tau=2e-3, b=4, tol=1e-12, maxit=8, r_max=40,
                                             seed=SEEDS["C1"])
    assert found2 and r2 == 9


def test_threshold_rank_not_found_by_rmax():
    op, s = _c1()
    res, r, found = oracle.lancsvd_threshold(op, tau=1e-6, b=4, tol=1e-12, maxit=8, r_max=6,
                                             seed=SEEDS["C1"])
    assert not found and r == 6 and len(res.S) == 6
    assert np.abs(res.S - s[:6]).max() / s[0] <= 1e-10
