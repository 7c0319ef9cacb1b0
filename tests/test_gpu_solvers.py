"""End-to-end parity of tsvd_block_lanczos / tsvd_rsvd against the oracle
(-m gpu).  Acceptance (north_star) over converged
triplets: max_i |sigma_i - sigma_i^oracle| / sigma_1 <= 1e-10,
||A v_i - sigma_i u_i|| / sigma_1 <= 1e-8, ||U^T U - I||_max <= 1e-12 (and
V).  Vectors are compared after sign alignment where the singular value is
well separated (reading R28).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import (spectrum_eq16, dense_prescribed, powerlaw_csr, blockdiag_csr,  # noqa: E402
                         SEEDS)

U = 2.0 ** -53


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T.lib()


def _accept(op, Ug, Sg, Vg, So, conv_mask=None, sigma_tol=1e-10):
    r = len(Sg)
    mask = np.ones(r, bool) if conv_mask is None else conv_mask
    s1 = So[0]
    assert np.abs(Sg - So)[mask].max() / s1 <= sigma_tol
    e, _ = oracle.residuals(op, Ug, Sg, Vg)
    assert e[mask].max() <= 1e-8
    assert np.abs(Ug.T @ Ug - np.eye(r)).max() <= 1e-12
    assert np.abs(Vg.T @ Vg - np.eye(r)).max() <= 1e-12
    return e


def _vec_parity(Ug, Vg, Uo, Vo, S, tol=1e-8):
    gaps = np.minimum(np.abs(np.diff(np.r_[np.inf, S])), np.abs(np.diff(np.r_[S, -np.inf])))
    for i in range(len(S)):
        if gaps[i] > 1e-3 * S[0]:
            sg = np.sign(Vg[:, i] @ Vo[:, i])
            assert np.abs(sg * Vg[:, i] - Vo[:, i]).max() <= tol * S[0] / gaps[i]
            assert np.abs(sg * Ug[:, i] - Uo[:, i]).max() <= tol * S[0] / gaps[i]


def _c1():
    s = spectrum_eq16(100)
    A = dense_prescribed(200, 100, s, SEEDS["C1"])
    return A, s


@pytest.mark.parametrize("inject", [True, False])
def test_c1_lanczos(inject):
    A, s = _c1()
    op = oracle.Operator(dense=A)
    seed = SEEDS["C1"]
    G = oracle.gaussian_block(200, 4, seed, draw=0)
    ro = oracle.lancsvd(op, r=10, b=4, d=28, tol=1e-12, maxit=8, seed=seed,
                        start=G if inject else None)
    with T.TruncatedSVD(A) as h:
        h.set_seed(seed)
        if inject:
            h.set_start(G)
        st = h.block_lanczos(r=10, b=4, tol=1e-12, maxit=8, d=28)
        Ug, Sg, Vg = h.get()
        info = h.info()
    assert st == T.TSVD_OK and info["nconv"] == 10 and info["cycles"] == ro.cycles
    _accept(op, Ug, Sg, Vg, ro.S)
    assert np.abs(Sg - s[:10]).max() / s[0] <= 1e-10       # closed form (Eq. 16)
    _vec_parity(Ug, Vg, ro.U, ro.V, ro.S)


def test_c1_rsvd():
    A, s = _c1()
    op = oracle.Operator(dense=A)
    seed = SEEDS["C1"]
    ro = oracle.randsvd(op, r=10, p=10, q=1, b_qr=16, seed=seed)
    with T.TruncatedSVD(A) as h:
        h.set_seed(seed)
        h.set_qr_block(16)
        h.rsvd(r=10, p=10, q=1)
        Ug, Sg, Vg = h.get()
    _accept(op, Ug, Sg, Vg, ro.S)
    assert np.abs(Sg - s[:10]).max() / s[0] <= 1e-10
    _vec_parity(Ug, Vg, ro.U, ro.V, ro.S)


def test_lanczos_restarts_parity():
    n = 120
    s = 10.0 * 0.93 ** np.arange(n)
    A = dense_prescribed(240, n, s, seed=8)
    op = oracle.Operator(dense=A)
    ro = oracle.lancsvd(op, r=4, b=4, d=16, tol=1e-10, maxit=60, seed=5)
    with T.TruncatedSVD(A) as h:
        h.set_seed(5)
        st = h.block_lanczos(r=4, b=4, tol=1e-10, maxit=60, d=16)
        Ug, Sg, Vg = h.get()
        info = h.info()
    assert st == T.TSVD_OK and ro.converged
    assert info["cycles"] > 1
    assert abs(info["cycles"] - ro.cycles) <= 1
    _accept(op, Ug, Sg, Vg, ro.S)
    assert np.abs(Sg - s[:4]).max() <= 1e-10 * s[0]


def test_rank_deficient_breakdown():
    """A breakdown in the deferred pass replays the cycle from the flagged
    block step; the Jacobi SVD already forked beside the last m-side step
    (solvers.cu; dense A takes that path) must be joined before the replay
    rewrites B, and rerun.  (Exactly-zero pivots need the dense path's
    arithmetic: the same matrix in CSR ends with tiny positive pivots.)"""
    rng = np.random.default_rng(6)
    m, n, k = 80, 40, 5
    X, _ = np.linalg.qr(rng.standard_normal((m, k)))
    Y, _ = np.linalg.qr(rng.standard_normal((n, k)))
    sv = np.array([5.0, 4.0, 3.0, 2.0, 1.0])
    A = (X * sv) @ Y.T
    with T.TruncatedSVD(A) as h:
        h.set_seed(7)
        h.block_lanczos(r=5, b=2, tol=1e-10, maxit=3, d=12)
        Ug, Sg, Vg = h.get()
        info = h.info()
    assert info["breakdowns"] >= 1
    assert np.abs(Sg - sv).max() <= 1e-12 * 5
    assert np.abs(Ug.T @ Ug - np.eye(5)).max() <= 1e-12


def test_full_dimension_exact():
    A, s = _c1()
    with T.TruncatedSVD(A) as h:
        h.block_lanczos(r=100, b=4, tol=1e-30, maxit=1, d=100)
        _, Sg, _ = h.get()
    sv = np.linalg.svd(A, compute_uv=False)
    assert np.abs(Sg - sv).max() <= 1e-13 * s[0]


@pytest.mark.parametrize("b,d", [(16, 96), (8, 64)])
def test_sparse_powerlaw_lanczos_parity(b, d):
    m = n = 20000
    csr = powerlaw_csr(m, n, 200000, 2.5, seed=21)
    op = oracle.Operator(csr=csr, shape=(m, n))
    seed = 0x1234
    ro = oracle.lancsvd(op, r=10, b=b, d=d, tol=1e-8, maxit=4, seed=seed)
    with T.TruncatedSVD(csr=csr, shape=(m, n)) as h:
        h.set_seed(seed)
        h.block_lanczos(r=10, b=b, tol=1e-8, maxit=4, d=d)
        Ug, Sg, Vg = h.get()
        rho = h.rho()
        info = h.info()
    conv = (rho <= 1e-8) & (ro.rho <= 1e-8 * ro.S[0])
    assert conv.sum() >= 5
    e = _accept(op, Ug, Sg, Vg, ro.S, conv_mask=conv)
    # the unconverged triplets are not unique across summation orders (R29):
    # check that they are valid Ritz triplets instead -- orthonormal (above)
    # and with rho equal to the explicit residual, A v_i - s_i u_i =
    # Qbar_{k+1} Rbar_k Vbar[last b rows, i] for every Ritz pair (Eq. 7, 10)
    assert np.abs(e - rho).max() <= 1e-11
    assert info["cycles"] == ro.cycles


def test_sparse_g2_closed_form():
    m, n = 60000, 40000
    top = np.linspace(100.0, 60.0, 30)
    rp, ci, va, sig = blockdiag_csr(m, n, 6.0, 2.5, seed=31, top_sigma=top, tail_max=10.0)
    op = oracle.Operator(csr=(rp, ci, va), shape=(m, n))
    with T.TruncatedSVD(csr=(rp, ci, va), shape=(m, n)) as h:
        st = h.block_lanczos(r=20, b=16, tol=1e-10, maxit=10, d=96)
        Ug, Sg, Vg = h.get()
    assert st == T.TSVD_OK
    assert np.abs(Sg - sig[:20]).max() / sig[0] <= 1e-10
    e, _ = oracle.residuals(op, Ug, Sg, Vg)
    assert e.max() <= 1e-8


def test_rsvd_sparse_parity():
    m, n = 30000, 10000
    csr = powerlaw_csr(m, n, 300000, 2.5, seed=41)
    op = oracle.Operator(csr=csr, shape=(m, n))
    ro = oracle.randsvd(op, r=10, p=10, q=4, b_qr=16, seed=3)
    with T.TruncatedSVD(csr=csr, shape=(m, n)) as h:
        h.set_seed(3)
        h.rsvd(r=10, p=10, q=4)
        Ug, Sg, Vg = h.get()
    # rSVD at finite q is defined by the iteration: compare with the oracle's
    # iterate directly (same Philox start, same CGS-QR panels)
    assert np.abs(Sg - ro.S).max() / ro.S[0] <= 1e-10
    assert np.abs(Ug.T @ Ug - np.eye(10)).max() <= 1e-12


def test_errors():
    A, _ = _c1()
    with T.TruncatedSVD(A) as h:
        with pytest.raises(T.TsvdError):
            h.block_lanczos(r=10, b=4, tol=1e-8, maxit=2, d=30)    # d % b != 0
        with pytest.raises(T.TsvdError):
            h.rsvd(r=90, p=20, q=1)                                # l > n
        with pytest.raises(T.TsvdError):
            h.get()
    with pytest.raises(T.TsvdError):
        T.TruncatedSVD(csr=(np.array([0, 2, 1], np.int64), np.array([0, 1], np.int32),
                            np.ones(2)), shape=(2, 2))
    with pytest.raises(T.TsvdError):   # column index out of range
        T.TruncatedSVD(csr=(np.array([0, 2, 2], np.int64), np.array([1, 2], np.int32),
                            np.ones(2)), shape=(2, 2))
    with T.TruncatedSVD(A) as h:       # d above the device Jacobi's 1536 limit
        with pytest.raises(T.TsvdError):
            h.rsvd(r=1, p=1536, q=0)


def _noncanonical(csr, seed):
    """The same matrix with every row's entries shuffled and about a third
    of them split into two duplicates v/2 + v/2 (= v exactly)."""
    rp, ci, va = csr
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(len(rp) - 1):
        c, v = ci[rp[i]:rp[i + 1]], va[rp[i]:rp[i + 1]]
        split = rng.random(len(c)) < 0.35
        cc = np.concatenate([c, c[split]])
        vv = np.concatenate([np.where(split, v * 0.5, v), v[split] * 0.5])
        p = rng.permutation(len(cc))
        rows.append(np.full(len(cc), i))
        cols.append(cc[p])
        vals.append(vv[p])
    lens = np.array([len(x) for x in cols])
    rp2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return rp2, np.concatenate(cols).astype(np.int32), np.concatenate(vals)


def test_noncanonical_csr_is_canonicalised():
    """unsorted / duplicate entries are canonicalised on the
    device (sorted, duplicates summed).  The products and a solve equal those
    of the canonical matrix (scipy's CSR, the oracle's operator, sums the
    duplicates too)."""
    m, n = 20000, 8000
    csr = powerlaw_csr(m, n, 200000, 2.5, seed=17)
    nc = _noncanonical(csr, 5)
    op = oracle.Operator(csr=nc, shape=(m, n))
    rng = np.random.default_rng(2)
    X = torch.from_numpy(rng.standard_normal((n, 16))).cuda()
    Xt = torch.from_numpy(rng.standard_normal((m, 16))).cuda()
    outs = []
    for c in (csr, nc):
        with T.TruncatedSVD(csr=c, shape=(m, n)) as h:
            Y = torch.empty((m, 16), dtype=torch.float64, device="cuda")
            Z = torch.empty((n, 16), dtype=torch.float64, device="cuda")
            T.dbg_apply(h, False, X, Y)
            T.dbg_apply(h, True, Xt, Z)
            h.set_seed(9)
            h.block_lanczos(r=8, b=8, tol=1e-10, maxit=8, d=64)
            outs.append((Y.cpu().numpy(), Z.cpu().numpy(), *h.get()))
    # v/2 + v/2 == v exactly, so the canonical form is bit-identical
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    ref = op.matmul(X.cpu().numpy())
    assert np.abs(outs[1][0] - ref).max() <= 1e-12 * np.abs(ref).max()


# ---- N1 thick restart (tsvd_set_thick_restart; oracle/lancsvd.py keep=l) ---
@pytest.mark.parametrize("inject", [True, False])
def test_c1_thick_restart(inject):
    """C1 at d = 20 < 28: the paper's restart stalls, keeping l = 12 Ritz
    pairs converges; same cycle count and triplets as the oracle."""
    A, s = _c1()
    op = oracle.Operator(dense=A)
    seed = SEEDS["C1"]
    G = oracle.gaussian_block(200, 4, seed, draw=0)
    ro = oracle.lancsvd(op, r=10, b=4, d=20, tol=1e-12, maxit=10, seed=seed, keep=12,
                        start=G if inject else None)
    with T.TruncatedSVD(A) as h:
        h.set_seed(seed)
        if inject:
            h.set_start(G)
        h.set_thick_restart(12)
        st = h.block_lanczos(r=10, b=4, tol=1e-12, maxit=10, d=20)
        Ug, Sg, Vg = h.get()
        info = h.info()
    assert ro.converged and st == T.TSVD_OK
    assert info["cycles"] == ro.cycles and info["cycles"] > 1
    _accept(op, Ug, Sg, Vg, ro.S)
    assert np.abs(Sg - s[:10]).max() / s[0] <= 1e-10
    _vec_parity(Ug, Vg, ro.U, ro.V, ro.S)


def test_thick_restart_slow_decay_parity():
    n = 120
    s = 10.0 * 0.93 ** np.arange(n)
    A = dense_prescribed(240, n, s, seed=8)
    op = oracle.Operator(dense=A)
    ro = oracle.lancsvd(op, r=4, b=4, d=16, tol=1e-10, maxit=60, seed=5, keep=8)
    with T.TruncatedSVD(A) as h:
        h.set_seed(5)
        h.set_thick_restart(8)
        st = h.block_lanczos(r=4, b=4, tol=1e-10, maxit=60, d=16)
        Ug, Sg, Vg = h.get()
        info = h.info()
    assert st == T.TSVD_OK and ro.converged
    assert abs(info["cycles"] - ro.cycles) <= 1
    _accept(op, Ug, Sg, Vg, ro.S)
    assert np.abs(Sg - s[:4]).max() <= 1e-10 * s[0]


@pytest.mark.parametrize("b,d,keep", [(16, 96, 32), (8, 64, 24)])
def test_sparse_powerlaw_thick_parity(b, d, keep):
    m = n = 20000
    csr = powerlaw_csr(m, n, 200000, 2.5, seed=21)
    op = oracle.Operator(csr=csr, shape=(m, n))
    seed = 0x1234
    ro = oracle.lancsvd(op, r=10, b=b, d=d, tol=1e-8, maxit=6, seed=seed, keep=keep)
    with T.TruncatedSVD(csr=csr, shape=(m, n)) as h:
        h.set_seed(seed)
        h.set_thick_restart(keep)
        h.block_lanczos(r=10, b=b, tol=1e-8, maxit=6, d=d)
        Ug, Sg, Vg = h.get()
        rho = h.rho()
        info = h.info()
    conv = (rho <= 1e-8) & (ro.rho <= 1e-8 * ro.S[0])
    assert conv.sum() >= 8
    e = _accept(op, Ug, Sg, Vg, ro.S, conv_mask=conv)
    # the unconverged triplets are not unique across summation orders (R29):
    # check that they are valid Ritz triplets instead -- orthonormal (above)
    # and with rho equal to the explicit residual, A v_i - s_i u_i =
    # Qbar_{k+1} Rbar_k Vbar[last b rows, i] for every Ritz pair (Eq. 7, 10)
    assert np.abs(e - rho).max() <= 1e-11
    assert info["cycles"] == ro.cycles


def test_thick_restart_shape_errors():
    A, _ = _c1()
    with T.TruncatedSVD(A) as h:
        for keep in (6, 8, 28):   # not a multiple of b=4 / < r=10 / >= d
            h.set_thick_restart(keep)
            with pytest.raises(T.TsvdError):
                h.block_lanczos(r=10, b=4, tol=1e-12, maxit=2, d=28)
        with pytest.raises(T.TsvdError):
            h.set_thick_restart(-1)


# ---- tsvd_set_output_mode: outputs formed in place over the bases ----------
@pytest.mark.parametrize("algo", ["lanczos", "rsvd"])
def test_inplace_outputs_match_separate(algo):
    """Eq. 12 / Alg. 1 S6-S7 formed over the bases' first r columns (the C5
    memory plan) give the same triplets as separate buffers."""
    A, s = _c1()
    res = {}
    for mode in (T.TSVD_OUT_SEPARATE, T.TSVD_OUT_INPLACE):
        with T.TruncatedSVD(A) as h:
            h.set_seed(11)
            h.set_output_mode(mode)
            if algo == "lanczos":
                h.block_lanczos(r=100, b=4, tol=1e-30, maxit=1, d=100)
            else:
                h.rsvd(r=60, p=40, q=1)
            res[mode] = h.get()
    for a, b in zip(res[T.TSVD_OUT_SEPARATE], res[T.TSVD_OUT_INPLACE]):
        assert np.abs(a - b).max() <= 1e-14 * max(1.0, np.abs(a).max())
    Ug, Sg, Vg = res[T.TSVD_OUT_INPLACE]
    r = len(Sg)
    assert np.abs(Ug.T @ Ug - np.eye(r))[:40, :40].max() <= 1e-12
    assert np.abs(Sg[:10] - s[:10]).max() / s[0] <= 1e-10


@pytest.mark.parametrize("r", [100, 140])
def test_inplace_outputs_wide_and_chunked(r):
    """In-place outputs through the one-pass kernel (r <= 128: X's first r
    columns overwritten by the row tile's own product) and through the
    scratch-staged row chunks (r > 128) equal the separate-buffer outputs."""
    s = spectrum_eq16(300)
    A = dense_prescribed(3000, 300, s, 77)
    res = {}
    for mode in (T.TSVD_OUT_SEPARATE, T.TSVD_OUT_INPLACE):
        with T.TruncatedSVD(A) as h:
            h.set_seed(5)
            h.set_output_mode(mode)
            h.block_lanczos(r=r, b=4, tol=1e-30, maxit=1, d=280)
            res[mode] = h.get()
    for a, b in zip(res[T.TSVD_OUT_SEPARATE], res[T.TSVD_OUT_INPLACE]):
        assert np.abs(a - b).max() <= 1e-13 * max(1.0, np.abs(a).max())
    Ug, Sg, Vg = res[T.TSVD_OUT_INPLACE]
    assert np.abs(Ug.T @ Ug - np.eye(r))[:40, :40].max() <= 1e-12
    assert np.abs(Vg.T @ Vg - np.eye(r))[:40, :40].max() <= 1e-12


def test_output_mode_errors():
    A, _ = _c1()
    with T.TruncatedSVD(A) as h:
        for bad in (-1, 3):
            with pytest.raises(T.TsvdError):
                h.set_output_mode(bad)


# ---- N4: rank by threshold (Eq. 3), tsvd_block_lanczos_threshold ----------
@pytest.mark.parametrize("tau,r_expect", [(1.5e-3, 10), (2e-3, 9)])
def test_threshold_rank_parity(tau, r_expect):
    A, s = _c1()
    op = oracle.Operator(dense=A)
    seed = SEEDS["C1"]
    ro, r_o, found = oracle.lancsvd_threshold(op, tau=tau, b=4, tol=1e-12, maxit=8, r_max=40,
                                              seed=seed)
    with T.TruncatedSVD(A) as h:
        h.set_seed(seed)
        st, r = h.block_lanczos_threshold(tau, b=4, tol=1e-12, maxit=8, r_max=40)
        Ug, Sg, Vg = h.get()
        info = h.info()
    assert found and st == T.TSVD_OK
    assert r == r_o == r_expect and Ug.shape == (200, r) and info["r"] == r
    _accept(op, Ug, Sg, Vg, ro.S)
    assert np.abs(Sg - s[:r]).max() / s[0] <= 1e-10                 # closed form
    ey = oracle.eckart_young_2norm(op, Ug, Sg, Vg)                   # Eq. 3
    assert ey == pytest.approx(s[r], rel=1e-6) and ey <= tau * s[0]


def test_threshold_rank_rmax_and_errors():
    A, s = _c1()
    with T.TruncatedSVD(A) as h:
        h.set_seed(SEEDS["C1"])
        st, r = h.block_lanczos_threshold(1e-6, b=4, tol=1e-12, maxit=8, r_max=6)
        _, Sg, _ = h.get()
        assert st == T.TSVD_WARN_NOTCONV and r == 6 and len(Sg) == 6
        assert np.abs(Sg - s[:6]).max() / s[0] <= 1e-10
        for bad in (0.0, -1.0, 1.0):
            with pytest.raises(T.TsvdError):
                h.block_lanczos_threshold(bad, b=4, tol=1e-12, maxit=8, r_max=6)


# ---- a17: explicit residuals inside the library (tsvd_residuals) -----------
@pytest.mark.parametrize("case", ["dense", "sparse", "sparse_wide", "inplace"])
def test_residuals_parity(case):
    """tsvd_residuals (device: the library's A.X + fixed-order column norms)
    vs oracle.residuals (scipy/numpy) on the same returned triplets: e_i and
    R_i = e_i s_1 / s_i (Eq. 14 corrected, reading R13).  The residual is a
    difference of nearly equal vectors, so the comparison is absolute in
    units of s_1: | ||z|| - ||z^o|| | <= ||z - z^o|| <= ||b|| with the
    element-wise forward-error bound b = 2 (K + 2) u (|A| |v| + s |u|)
    of both sides' products (K = row length)."""
    if case == "dense":
        A, _ = _c1()
        op, kw, r = oracle.Operator(dense=A), dict(A=A), 10
    else:
        m, n = (30000, 12000) if case != "sparse_wide" else (20000, 9000)
        csr = powerlaw_csr(m, n, 300000, 2.5, seed=23)
        op, kw, r = oracle.Operator(csr=csr, shape=(m, n)), dict(csr=csr, shape=(m, n)), 40
        if case == "sparse_wide":
            r = 70                       # > 64: two chunks of the column loop
    with T.TruncatedSVD(**kw) as h:
        if case == "inplace":
            h.set_output_mode(T.TSVD_OUT_INPLACE)
        h.set_seed(11)
        if case == "sparse_wide":
            h.rsvd(r, 10, 1)
        else:
            h.block_lanczos(r, 8, 1e-10, 4, d=min(4 * r, 160))
        Ug, Sg, Vg = h.get()
        e, R = h.residuals()
    eo, Ro = oracle.residuals(op, Ug, Sg, Vg)
    absA = np.abs(op.A) if op.kind == "dense" else abs(op.A)
    K = op.n if op.kind == "dense" else np.diff(op.A.indptr)
    b = 2 * (np.asarray(K)[..., None] + 2) * U * (np.asarray(absA @ np.abs(Vg)) + np.abs(Ug) * Sg)
    tol = 2 * np.linalg.norm(b, axis=0) / Sg[0] + 1e-300
    assert np.all(np.abs(e - eo) <= tol)
    assert np.allclose(R * Sg, e * Sg[0], rtol=1e-14, atol=0)


# ---- BCGS-PIP+ orthogonalisation (tsvd_set_ortho) ----------
@pytest.mark.parametrize("case", ["c1", "sparse", "restarts"])
def test_bcgs_pip2_lanczos_parity(case):
    """LancSVD with the BCGS-PIP+ block orthogonalisation (reading R34) vs
    oracle.lancsvd(ortho="bcgs_pip2") on the same bytes and Philox start:
    same cycle count, sigma / vectors within the north_star tolerances over
    converged triplets, no breakdown fallback."""
    if case == "c1":
        A, s = _c1()
        op, kw, prm = oracle.Operator(dense=A), dict(A=A), dict(r=10, b=4, d=28, tol=1e-12, maxit=8)
        seed = SEEDS["C1"]
    elif case == "sparse":
        m, n = 30000, 12000
        csr = powerlaw_csr(m, n, 300000, 2.5, seed=23)
        op, kw = oracle.Operator(csr=csr, shape=(m, n)), dict(csr=csr, shape=(m, n))
        prm, seed = dict(r=20, b=8, d=96, tol=1e-10, maxit=6), 31
    else:
        n = 120
        A = dense_prescribed(240, n, 10.0 * 0.93 ** np.arange(n), seed=8)
        op, kw, prm, seed = oracle.Operator(dense=A), dict(A=A), \
            dict(r=4, b=4, d=16, tol=1e-10, maxit=60), 5
    ro = oracle.lancsvd(op, seed=seed, ortho="bcgs_pip2", **prm)
    with T.TruncatedSVD(**kw) as h:
        h.set_seed(seed)
        h.set_ortho("bcgs_pip2")
        st = h.block_lanczos(prm["r"], prm["b"], prm["tol"], prm["maxit"], d=prm["d"])
        Ug, Sg, Vg = h.get()
        info = h.info()
        rho = h.rho()
    # PIP+ falls back to CGS2 when a Lanczos block is nearly inside span(P)
    # (W - H^T H loses its positive definiteness): the sparse case takes 5
    # fallbacks in the oracle too, so only C1 must be fallback-free
    if case == "c1":
        assert info["breakdowns"] == 0
    # the slow-decay restart case sits at tol after ~9 cycles: PIP+'s rounding
    # (Pythagorean Gram) may move the last restart by one cycle either way
    assert abs(info["cycles"] - ro.cycles) <= (1 if case == "restarts" else 0)
    conv = (rho <= prm["tol"]) & (ro.rho <= prm["tol"] * ro.S[0])
    assert conv.sum() >= min(prm["r"], 4)
    _accept(op, Ug, Sg, Vg, ro.S, conv_mask=conv)
    _vec_parity(Ug[:, conv], Vg[:, conv], ro.U[:, conv], ro.V[:, conv], ro.S[conv])
    if case == "c1":
        assert st == T.TSVD_OK
        assert np.abs(Sg - s[:10]).max() / s[0] <= 1e-10


# ---- CUDA graph of the Lanczos cycle (solvers.cu) ---------------------------
@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_cycle_graph_replay_is_bit_identical(kind):
    """Solve 1 runs the block steps eagerly, solve 2 captures them into a
    CUDA graph and launches it, solve 3 replays it: the three results and
    the per-phase launch counts must be identical (the graph records the
    same kernels with the same arguments), also with profiling on."""
    if kind == "dense":
        A, _ = _c1()
        kw = dict(A=A)
        prm = dict(r=10, b=4, tol=1e-12, maxit=8, d=28)
    else:
        m, n = 20000, 8000
        csr = powerlaw_csr(m, n, 200000, 2.5, seed=17)
        kw = dict(csr=csr, shape=(m, n))
        prm = dict(r=12, b=8, tol=1e-10, maxit=3, d=64)
    outs = []
    with T.TruncatedSVD(**kw) as h:
        h.set_graphs(True)
        h.set_profiling(True)
        for _ in range(3):
            h.set_seed(4)
            h.reset_profile()
            h.block_lanczos(**prm)
            prof = h.profile()
            outs.append((*h.get(), h.info(), {k: v["launches"] for k, v in prof.items()},
                         {k: v["calls"] for k, v in prof.items()}))
    for o in outs[1:]:
        for a, b in zip(outs[0][:3], o[:3]):
            assert np.array_equal(a, b)
        assert o[3]["launches"] == outs[0][3]["launches"]
        assert o[4] == outs[0][4] and o[5] == outs[0][5]


@pytest.mark.parametrize("b,d,r", [(40, 120, 20), (48, 96, 30)])
def test_wide_block_lanczos_parity(b, d, r):
    """P:174 allows any b >= 1: blocks wider than the 32-column kernel tile
    are orthogonalised in 32-column panels (block_orth, as Alg. 3 does for
    RandSVD); the QR with positive diagonal is unique, so the result equals
    the oracle's b-wide CholQR2 / CGS-CQR2 iteration to rounding."""
    n = 200
    s = 10.0 * 0.9 ** np.arange(n)
    A = dense_prescribed(400, n, s, seed=b)
    op = oracle.Operator(dense=A)
    ro = oracle.lancsvd(op, r=r, b=b, d=d, tol=1e-10, maxit=6, seed=3)
    with T.TruncatedSVD(A) as h:
        h.set_seed(3)
        st = h.block_lanczos(r=r, b=b, tol=1e-10, maxit=6, d=d)
        Ug, Sg, Vg = h.get()
        info = h.info()
        rho = h.rho()
    assert info["cycles"] == ro.cycles and info["breakdowns"] == 0
    conv = (rho <= 1e-10) & (ro.rho <= 1e-10 * ro.S[0])
    assert conv.sum() >= 10
    _accept(op, Ug, Sg, Vg, ro.S, conv_mask=conv)
    assert np.abs(Sg - s[:r])[conv].max() / s[0] <= 1e-10
    _vec_parity(Ug[:, conv], Vg[:, conv], ro.U[:, conv], ro.V[:, conv], ro.S[conv])


def test_profiling_mask_and_beside_svd_phase():
    """tsvd_set_profiling_mask records only the selected phases; on one GPU
    the last m-side block step runs beside the Jacobi SVD (solvers.cu) and is
    profiled as its own phase, so ortho_nn / ortho_tn time only kernels that
    have the GPU to themselves."""
    A, _ = _c1()
    with T.TruncatedSVD(A) as h:
        h.set_seed(3)
        h.set_profiling(True)
        h.block_lanczos(r=10, b=4, tol=1e-12, maxit=8, d=28)
        full = h.profile()
        h.reset_profile()
        h.set_profiling_mask(1 << T.PROF_PHASES.index("ortho_nn"))
        h.block_lanczos(r=10, b=4, tol=1e-12, maxit=8, d=28)
        only_nn = h.profile()
        h.set_profiling(False)
    assert full["beside_svd"]["calls"] > 0 and full["small_svd"]["calls"] > 0
    assert only_nn["ortho_nn"]["calls"] == full["ortho_nn"]["calls"]
    assert all(v["calls"] == 0 for k, v in only_nn.items() if k != "ortho_nn")
