"""Kernel-level parity: each CUDA building block against the oracle on the
same seeded inputs (-m gpu, through the C ABI's tsvd_dbg_* entry points).

Tolerances: products use the forward-error bound |y - y_ref| <= c*K*u*sum|a||x|
(K = reduction length); orthogonalisation results are compared elementwise
with a bound proportional to u * cond (the forward error of a QR factor);
Philox words bit-exact; normals within a few ulp (CUDA vs glibc log/cos).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle.core import DrawCtx  # noqa: E402
from oracle.philox import philox4x32_10, gaussian_block  # noqa: E402
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import powerlaw_csr  # noqa: E402

U = 2.0 ** -53


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T.lib()


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_philox_words_bit_exact():
    rng = np.random.default_rng(0)
    n = 4096
    ctr = rng.integers(0, 2 ** 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0
    key[0] = 0
    ctr[1] = 0xFFFFFFFF
    key[1] = 0xFFFFFFFF
    out = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
    T.dbg_philox_words(cu(ctr.view(np.int32)), cu(key.view(np.int32)), out)
    got = out.cpu().numpy().view(np.uint32)
    ref = philox4x32_10(tuple(ctr[:, i].astype(np.uint64) for i in range(4)),
                        (key[:, 0].astype(np.uint64), key[:, 1].astype(np.uint64)))
    ref = np.stack([r.astype(np.uint32) for r in ref], axis=1)
    assert np.array_equal(got, ref)
    assert [hex(x) for x in got[0]] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]


@pytest.mark.parametrize("q,w,row0,qt,draw", [(1000, 4, 0, 1000, 0), (777, 16, 123, 5000, 3),
                                              (64, 1, 0, 64, 9)])
def test_philox_normal_ulp(q, w, row0, qt, draw):
    seed = 0x2403062181
    out = torch.empty((q, w), dtype=torch.float64, device="cuda")
    T.dbg_philox(out, seed, draw, row0, qt)
    ref = gaussian_block(q, w, seed, draw=draw, row0=row0, q_total=qt)
    got = out.cpu().numpy()
    assert np.abs(got - ref).max() <= 8 * U * np.abs(ref).max()


@pytest.mark.parametrize("q,s,w", [(1, 1, 1), (100, 7, 3), (1000, 33, 16), (4097, 130, 32),
                                   (200000, 64, 16), (3000, 10, 40), (129, 300, 8),
                                   (100000, 300, 32), (5000, 20, 28), (64001, 16, 32),
                                   (30000, 640, 24)])
def test_gemm_tn(q, s, w):
    rng = np.random.default_rng(q + s + w)
    X = rng.standard_normal((q, s))
    Y = rng.standard_normal((q, w))
    Cg = torch.zeros((s, w), dtype=torch.float64, device="cuda")
    T.dbg_gemm_tn(cu(X), cu(Y), Cg)
    ref = X.T @ Y
    bound = 4 * q * U * (np.abs(X).T @ np.abs(Y)) + 1e-300
    assert np.all(np.abs(Cg.cpu().numpy() - ref) <= bound)


@pytest.mark.parametrize("q,s,w,alpha,beta", [(1, 1, 1, 1.0, 0.0), (100, 7, 3, -1.0, 1.0),
                                              (4097, 130, 32, -1.0, 1.0), (1000, 0, 16, 0.0, 1.0),
                                              (3000, 50, 40, 1.0, 0.0), (65, 700, 8, 2.0, 0.5),
                                              (50000, 320, 32, -1.0, 1.0), (20001, 96, 24, 1.0, 0.0),
                                              (777, 40, 18, 0.5, -2.0), (9000, 2000, 32, 1.0, 0.0),
                                              (5000, 0, 32, 0.0, 1.0), (3001, 0, 24, 0.0, -0.5),
                                              (200000, 40, 32, -1.0, 1.0), (150000, 20, 32, 1.0, 1.0)])
def test_gemm_nn(q, s, w, alpha, beta):
    rng = np.random.default_rng(q * 7 + s + w)
    X = rng.standard_normal((q, max(s, 1)))[:, :s]
    H = rng.standard_normal((max(s, 1), w))[:s]
    Z0 = rng.standard_normal((q, w))
    Zg = cu(Z0)
    T.dbg_gemm_nn(cu(X) if s else cu(np.zeros((q, 1))), cu(H) if s else cu(np.zeros((1, w))),
                  Zg, alpha, beta)
    ref = beta * Z0 + alpha * (X @ H)
    bound = 4 * (s + 2) * U * (abs(beta) * np.abs(Z0) + abs(alpha) * np.abs(X) @ np.abs(H)) + 1e-300
    assert np.all(np.abs(Zg.cpu().numpy() - ref) <= bound)


def _csr_case(kind):
    if kind == "powerlaw":
        m, n = 30000, 20000
        rp, ci, va = powerlaw_csr(m, n, 400000, 2.5, seed=11)
    elif kind == "diag":
        m = n = 5000
        rp = np.arange(n + 1, dtype=np.int64)
        ci = np.arange(n, dtype=np.int32)
        va = np.random.default_rng(1).standard_normal(n)
    else:  # empty rows, one dense row, one very long column
        m, n = 9000, 8000
        rng = np.random.default_rng(5)
        rows = []
        for i in range(m):
            if i % 3 == 0:
                rows.append(np.array([], dtype=np.int64))
            elif i == 7:
                rows.append(np.arange(n))                       # dense row (split segments)
            else:
                rows.append(np.unique(np.concatenate([[0], rng.integers(0, n, 5)])))
        rp = np.zeros(m + 1, dtype=np.int64)
        rp[1:] = np.cumsum([len(r) for r in rows])
        ci = np.concatenate(rows).astype(np.int32)
        va = rng.standard_normal(len(ci))
    return (m, n), (rp, ci, va)


@pytest.mark.parametrize("kind", ["powerlaw", "diag", "edge"])
@pytest.mark.parametrize("w", [1, 4, 16, 32, 50])
def test_spmm_parity(kind, w):
    shape, csr = _csr_case(kind)
    m, n = shape
    op = oracle.Operator(csr=csr, shape=shape)
    h = T.TruncatedSVD(csr=csr, shape=shape)
    rng = np.random.default_rng(w)
    X = rng.standard_normal((n, w))
    Xt = rng.standard_normal((m, w))
    # NaN-filled outputs: every row (empty rows included) must be written
    Yg = torch.full((m, w), float("nan"), dtype=torch.float64, device="cuda")
    Zg = torch.full((n, w), float("nan"), dtype=torch.float64, device="cuda")
    T.dbg_apply(h, False, cu(X), Yg)
    T.dbg_apply(h, True, cu(Xt), Zg)
    Aabs = oracle.Operator(csr=(csr[0], csr[1], np.abs(csr[2])), shape=shape)
    ref, reft = op.matmul(X), op.rmatmul(Xt)
    rowlen = np.diff(csr[0]).max() + 1
    b1 = 2 * rowlen * U * Aabs.matmul(np.abs(X)) + 1e-300
    b2 = 2 * m * U * Aabs.rmatmul(np.abs(Xt)) + 1e-300
    assert np.all(np.abs(Yg.cpu().numpy() - ref) <= b1)
    assert np.all(np.abs(Zg.cpu().numpy() - reft) <= b2)
    if kind == "diag":
        assert np.array_equal(Yg.cpu().numpy(), ref)
    h.close()


@pytest.mark.parametrize("m,n,ws", [(3000, 1100, (4, 12, 32, 37)), (20000, 2500, (16, 29, 69)),
                                    (41000, 700, (32, 64))])
def test_dense_apply_parity(m, n, ws):
    """Dense A.X / A^T.X; few row tiles -> split-K partials summed in order."""
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n))
    h = T.TruncatedSVD(A)
    for w in ws:
        X = rng.standard_normal((n, w))
        Xt = rng.standard_normal((m, w))
        Yg = torch.zeros((m, w), dtype=torch.float64, device="cuda")
        Zg = torch.zeros((n, w), dtype=torch.float64, device="cuda")
        T.dbg_apply(h, False, cu(X), Yg)
        T.dbg_apply(h, True, cu(Xt), Zg)
        assert np.all(np.abs(Yg.cpu().numpy() - A @ X) <= 4 * n * U * np.abs(A) @ np.abs(X))
        assert np.all(np.abs(Zg.cpu().numpy() - A.T @ Xt) <= 4 * m * U * np.abs(A.T) @ np.abs(Xt))
    h.close()


def _cond_matrix(q, w, kappa, rng):
    X, _ = np.linalg.qr(rng.standard_normal((q, w)))
    Y, _ = np.linalg.qr(rng.standard_normal((w, w)))
    return (X * np.logspace(0, -np.log10(kappa), w)) @ Y.T


@pytest.mark.parametrize("q,w,kappa", [(100, 4, 10.0), (5000, 16, 1e6), (70001, 32, 1e3),
                                       (333, 7, 1e7), (9000, 23, 1e5), (12345, 31, 1e6),
                                       (3000, 32, 1e7)])
def test_cholqr2_parity(q, w, kappa):
    rng = np.random.default_rng(q + w)
    Y = _cond_matrix(q, w, kappa, rng) * 3.0
    Qo, Ro = oracle.cholqr2(Y, DrawCtx(1))
    Yg = cu(Y)
    Rg = torch.zeros((w, w), dtype=torch.float64, device="cuda")
    fb = T.dbg_cholqr2(Yg, Rg, seed=1)
    assert not fb  # kappa <= 1e7: no Cholesky breakdown (u kappa^2 < 1)
    Q, R = Yg.cpu().numpy(), Rg.cpu().numpy()
    assert np.abs(Q.T @ Q - np.eye(w)).max() <= 10 * w * U
    assert np.linalg.norm(Y - Q @ R) / np.linalg.norm(Y) <= 100 * U
    assert np.abs(Q - Qo).max() <= 1e-13 * kappa
    assert np.abs(R - Ro).max() <= 1e-13 * kappa * np.abs(Ro).max()


@pytest.mark.parametrize("q,s,w,kappa", [(1000, 8, 4, 1.0), (20000, 100, 16, 1e4),
                                         (4099, 37, 32, 1e7), (50000, 384, 16, 1e2),
                                         (30000, 320, 32, 1e3), (7000, 50, 27, 1e4),
                                         # many 128-row tiles per CTA with fewer K chunks
                                         # than ring stages (w = 32 folded producer)
                                         (200000, 32, 32, 1e2), (300000, 60, 32, 1e3)])
def test_cgs_cqr2_parity(q, s, w, kappa):
    rng = np.random.default_rng(q + s)
    P, _ = np.linalg.qr(rng.standard_normal((q, s)))
    Y = P @ rng.standard_normal((s, w)) + 1e-3 * _cond_matrix(q, w, kappa, rng)
    Qo, Ho, Ro = oracle.cgs_cqr2(Y, P, DrawCtx(2))
    basis = cu(np.hstack([P, Y]))
    Hg = torch.zeros((s, w), dtype=torch.float64, device="cuda")
    Rg = torch.zeros((w, w), dtype=torch.float64, device="cuda")
    fb = T.dbg_cgs_cqr2(basis, s, w, Hg, Rg, seed=2)
    assert not fb
    B = basis.cpu().numpy()
    Q, H, R = B[:, s:], Hg.cpu().numpy(), Rg.cpu().numpy()
    assert np.array_equal(B[:, :s], P)          # P untouched
    assert np.abs(P.T @ Q).max() <= 100 * U
    assert np.abs(Q.T @ Q - np.eye(w)).max() <= 10 * w * U
    assert np.linalg.norm(Y - P @ H - Q @ R) / np.linalg.norm(Y) <= 100 * U
    cond = np.linalg.cond(np.hstack([P, Y]))
    assert np.abs(Q - Qo).max() <= 1e-14 * cond
    assert np.abs(H - Ho).max() <= 1e-14 * cond * np.abs(Ho).max()
    assert np.abs(R - Ro).max() <= 1e-14 * cond * np.abs(Ro).max()


def test_breakdown_fallback_parity():
    rng = np.random.default_rng(4)
    q = 600
    P, _ = np.linalg.qr(rng.standard_normal((q, 5)))
    a = rng.standard_normal(q)
    # exactly zero remainder columns: Cholesky pivots exactly 0 on both sides
    Y = np.stack([a, np.zeros(q), P[:, 1] * 2.0, rng.standard_normal(q)], axis=1)
    Qo, Ho, Ro = oracle.cgs_cqr2(Y, P, DrawCtx(7))
    basis = cu(np.hstack([P, Y]))
    Hg = torch.zeros((5, 4), dtype=torch.float64, device="cuda")
    Rg = torch.zeros((4, 4), dtype=torch.float64, device="cuda")
    assert T.dbg_cgs_cqr2(basis, 5, 4, Hg, Rg, seed=7)   # fallback taken
    Q, H, R = basis.cpu().numpy()[:, 5:], Hg.cpu().numpy(), Rg.cpu().numpy()
    assert np.abs(Q.T @ Q - np.eye(4)).max() < 1e-14
    assert np.abs(P.T @ Q).max() < 1e-14
    assert np.linalg.norm(Y - P @ H - Q @ R) / np.linalg.norm(Y) < 1e-14
    assert R[1, 1] == 0.0 and Ro[1, 1] == 0.0
    # same Philox replacement draws on both sides
    assert np.abs(Q - Qo).max() < 1e-12
    assert np.abs(R - Ro).max() < 1e-12 and np.abs(H - Ho).max() < 1e-12


@pytest.mark.parametrize("q,l,bq", [(2000, 20, 16), (10000, 110, 16), (500, 37, 8)])
def test_cgs_qr_parity(q, l, bq):
    rng = np.random.default_rng(l)
    Y = _cond_matrix(q, l, 1e5, rng)
    Qo, Ro = oracle.cgs_qr(Y, bq, DrawCtx(0))
    Yg = cu(Y)
    Rg = torch.zeros((l, l), dtype=torch.float64, device="cuda")
    T.dbg_cgs_qr(Yg, bq, Rg)
    Q, R = Yg.cpu().numpy(), Rg.cpu().numpy()
    assert np.abs(Q.T @ Q - np.eye(l)).max() <= 1e-14
    assert np.linalg.norm(Y - Q @ R) / np.linalg.norm(Y) <= 1e-14
    assert np.abs(R - Ro).max() <= 1e-9 * np.abs(Ro).max()
    assert np.abs(Q - Qo).max() <= 1e-9


def _lanczos_like_B(d, b, rng):
    """Lower block-bidiagonal d x d with b x b blocks (Eq. 8) whose values
    follow a Lanczos B_k's: lower-triangular diagonal blocks L_i and upper
    triangular subdiagonal blocks Rbar_i with geometrically decaying norms."""
    B = np.zeros((d, d))
    k = d // b
    for i in range(k):
        sc = 100.0 * 0.97 ** i
        B[i * b:(i + 1) * b, i * b:(i + 1) * b] = sc * np.tril(rng.standard_normal((b, b)))
        if i + 1 < k:
            B[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = 0.3 * sc * np.triu(
                rng.standard_normal((b, b)))
    return B


@pytest.mark.parametrize("d,kind", [(1, "tri"), (5, "tri"), (28, "tri"), (64, "tri"),
                                    (97, "tri"), (200, "tri"), (384, "tri"), (513, "tri"),
                                    (384, "lanczos16"), (640, "lanczos32"),
                                    (704, "lanczos32"), (768, "tri"), (1024, "lanczos32"),
                                    (1536, "tri"), (1536, "lanczos32")])
def test_small_svd_parity(d, kind):
    """Device Jacobi vs LAPACK gesvd up to the largest d the library takes
    (C3: 640, C4: 704, limit 1536), on random lower-triangular B and on
    Lanczos-shaped block-bidiagonal B; the sweep cap is never hit."""
    rng = np.random.default_rng(d)
    if kind == "tri":
        B = np.tril(rng.standard_normal((d, d))) - np.tril(rng.standard_normal((d, d)), -5)
    else:
        B = _lanczos_like_B(d, int(kind[7:]), rng)
    Uo, So, Vo = oracle.small_svd(B)
    Ub = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    Vb = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    S = torch.zeros(d, dtype=torch.float64, device="cuda")
    sweeps = T.dbg_small_svd(cu(B), Ub, S, Vb)
    assert sweeps < 60
    Ug, Sg, Vg = Ub.cpu().numpy(), S.cpu().numpy(), Vb.cpu().numpy()
    tol = 10 * d * U * So[0]
    assert np.abs(Sg - So).max() <= tol
    assert np.all(np.diff(Sg) <= 0)
    assert np.abs(Ug @ np.diag(Sg) @ Vg.T - B).max() <= tol
    assert np.abs(Vg.T @ Vg - np.eye(d)).max() <= 10 * d * U
    # vectors up to sign where the singular value is simple
    gaps = np.minimum(np.abs(np.diff(np.r_[np.inf, So])), np.abs(np.diff(np.r_[So, -np.inf])))
    for i in range(d):
        if gaps[i] > 1e-6 * So[0]:
            sgn = np.sign(Vg[:, i] @ Vo[:, i])
            assert np.abs(sgn * Vg[:, i] - Vo[:, i]).max() <= 1e-10 * So[0] / gaps[i]
