"""Parity at BASELINE.json's full sizes for configs C3 (sparse rectangular,
LancSVD vs RandSVD q=2) and C4 (dense 40000 x 20000, Eq. 16 spectrum), in
the launch configuration bench.py times (-m gpu).

The oracle cannot run these solves in seconds, so (as in test_gpu_fullsize):
  * sampled outputs of the products are recomputed by the oracle one by one
    (rows of A.X and A^T.X at the configs' widths, forward-error bounds);
  * the solves are checked through properties that hold at any size:
      - LancSVD: the oracle's residual e_i = ||A v_i - s_i u_i|| / s_1,
        orthogonality, rho (Eq. 10) = explicit residual;
      - RandSVD: A^T U = V Sigma holds to rounding for Alg. 1's outputs
        (U = Qbar Vbar, V = Q Ubar, A^T Qbar = Q R_p => A^T U = Q R_p Vbar
        = Q Ubar Sigma = V Sigma), orthogonality;
      - C4: the spectrum is prescribed (Eq. 15/16, reading R14), so every
        converged sigma_i is pinned by Weyl's bound |s_i - sigma_i| <=
        ||A v_i - s_i u_i|| + ||A^T u_i - s_i v_i|| and, beyond that, to the
        north_star's 1e-10 sigma_1 for triplets converged to tol.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import oracle  # noqa: E402
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import CONFIGS, SEEDS, dense_prescribed, powerlaw_csr, spectrum_eq16  # noqa: E402

U = 2.0 ** -53


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def c3():
    _cuda()
    cfg = CONFIGS["C3"]
    csr = powerlaw_csr(cfg["m"], cfg["n"], cfg["nnz"], cfg["alpha"], SEEDS["C3"])
    dev = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in csr)
    op = oracle.Operator(csr=csr, shape=(cfg["m"], cfg["n"]))
    return cfg, csr, dev, op


@pytest.fixture(scope="module")
def c4():
    _cuda()
    cfg = CONFIGS["C4"]
    sig = spectrum_eq16(cfg["n"])
    A = dense_prescribed(cfg["m"], cfg["n"], sig, SEEDS["C4"], n_reflectors=4)
    return cfg, A, torch.from_numpy(A).cuda(), np.sort(sig)[::-1]


def _sampled_rows_check(Yh, X, rows_of, rows):
    for i in rows:
        cols, vals = rows_of(i)
        ref = vals @ X[cols]
        bound = 2 * (len(cols) + 1) * U * (np.abs(vals) @ np.abs(X[cols])) + 1e-300
        assert np.all(np.abs(Yh[i] - ref) <= bound), i


@pytest.mark.parametrize("w", [32, 110])
def test_c3_products_sampled(c3, w):
    """A.X and A^T.X at the LancSVD (b = 32) and RandSVD (l = 110) widths."""
    cfg, csr, dev, op = c3
    m, n = cfg["m"], cfg["n"]
    rp, ci, va = csr
    rng = np.random.default_rng(w)
    X = rng.standard_normal((n, w))
    Xt = rng.standard_normal((m, w))
    Y = torch.empty((m, w), dtype=torch.float64, device="cuda")
    Z = torch.empty((n, w), dtype=torch.float64, device="cuda")
    with T.TruncatedSVD(csr=dev, shape=(m, n)) as h:
        T.dbg_apply(h, False, torch.from_numpy(X).cuda(), Y)
        T.dbg_apply(h, True, torch.from_numpy(Xt).cuda(), Z)
    Yh, Zh = Y.cpu().numpy(), Z.cpu().numpy()
    lens = np.diff(rp)
    rows = np.unique(np.concatenate([rng.integers(0, m, 200), np.argsort(lens)[-10:],
                                     np.where(lens == 0)[0][:5]]))
    _sampled_rows_check(Yh, X, lambda i: (ci[rp[i]:rp[i + 1]], va[rp[i]:rp[i + 1]]), rows)
    AT = op.A.T.tocsr()
    cl = np.diff(AT.indptr)
    cols = np.unique(np.concatenate([rng.integers(0, n, 200), np.argsort(cl)[-10:]]))
    _sampled_rows_check(Zh, Xt, lambda j: (AT.indices[AT.indptr[j]:AT.indptr[j + 1]],
                                           AT.data[AT.indptr[j]:AT.indptr[j + 1]]), cols)


def test_c3_lanczos_properties(c3):
    cfg, csr, dev, op = c3
    m, n, r = cfg["m"], cfg["n"], cfg["r"]
    with T.TruncatedSVD(csr=dev, shape=(m, n)) as h:
        h.set_seed(SEEDS["C3"])
        st = h.block_lanczos(r, cfg["b"], cfg["tol"], cfg["maxit"], d=cfg["d"])
        Ug, Sg, Vg = h.get()
        rho = h.rho()
    conv = rho <= cfg["tol"]
    assert st == T.TSVD_OK          # all r = 100 converge (2 cycles at d = 640)
    assert conv.all()
    e, _ = oracle.residuals(op, Ug, Sg, Vg)
    assert e[conv].max() <= 1e-8
    assert np.abs(rho - e).max() <= 1e-12
    assert np.abs(Ug.T @ Ug - np.eye(r)).max() <= 1e-12
    assert np.abs(Vg.T @ Vg - np.eye(r)).max() <= 1e-12
    assert np.all(np.diff(Sg) <= 0)


def test_c3_rsvd_properties(c3):
    """RandSVD q = 2 (the C3 comparison): A^T U = V Sigma to rounding."""
    cfg, csr, dev, op = c3
    m, n, r = cfg["m"], cfg["n"], cfg["r"]
    with T.TruncatedSVD(csr=dev, shape=(m, n)) as h:
        h.set_seed(SEEDS["C3"])
        h.rsvd(r, cfg["rsvd_p"], cfg["rsvd_q"])
        Ug, Sg, Vg = h.get()
    assert np.abs(Ug.T @ Ug - np.eye(r)).max() <= 1e-12
    assert np.abs(Vg.T @ Vg - np.eye(r)).max() <= 1e-12
    assert np.all(np.diff(Sg) <= 0) and Sg[-1] > 0
    ATU = op.rmatmul(Ug)
    f = np.linalg.norm(ATU - Vg * Sg, axis=0) / Sg[0]
    assert f.max() <= 1e-11
    # Rayleigh-Ritz: U^T A V = Sigma (Alg. 1 S5-S7: U = Qbar Vbar, V = Q Ubar,
    # Qbar^T A Q = R_p^T), so sigma_i = u_i^T A v_i to rounding
    AV = op.matmul(Vg)
    assert np.abs(np.einsum("ij,ij->j", Ug, AV) - Sg).max() / Sg[0] <= 1e-12
    # residuals: ||A v - s u|| <= ||A v|| <= s_1 (parity with the oracle's
    # iterate: tests/test_gpu_oracle_fullsize.py::test_c3_rsvd_vs_oracle)
    e, _ = oracle.residuals(op, Ug, Sg, Vg)
    assert np.all(np.isfinite(e)) and e.max() <= 1.0 + 1e-12


def test_c4_products_sampled(c4):
    cfg, A, Ad, _ = c4
    m, n, w = cfg["m"], cfg["n"], cfg["b"]
    rng = np.random.default_rng(4)
    X = rng.standard_normal((n, w))
    Xt = rng.standard_normal((m, w))
    Y = torch.empty((m, w), dtype=torch.float64, device="cuda")
    Z = torch.empty((n, w), dtype=torch.float64, device="cuda")
    with T.TruncatedSVD(Ad) as h:
        T.dbg_apply(h, False, torch.from_numpy(X).cuda(), Y)
        T.dbg_apply(h, True, torch.from_numpy(Xt).cuda(), Z)
    Yh, Zh = Y.cpu().numpy(), Z.cpu().numpy()
    rows = rng.integers(0, m, 200)
    ref = A[rows] @ X
    bound = 2 * (n + 1) * U * (np.abs(A[rows]) @ np.abs(X))
    assert np.all(np.abs(Yh[rows] - ref) <= bound)
    cols = rng.integers(0, n, 200)
    reft = A[:, cols].T @ Xt
    boundt = 2 * (m + 1) * U * (np.abs(A[:, cols]).T @ np.abs(Xt))
    assert np.all(np.abs(Zh[cols] - reft) <= boundt)


def test_c4_lanczos_closed_form(c4):
    cfg, A, Ad, sig = c4
    r = cfg["r"]
    with T.TruncatedSVD(Ad) as h:
        h.set_seed(SEEDS["C4"])
        st = h.block_lanczos(r, cfg["b"], cfg["tol"], cfg["maxit"], d=cfg["d"])
        Ug, Sg, Vg = h.get()
        rho = h.rho()
    assert st in (T.TSVD_OK, T.TSVD_WARN_NOTCONV)
    conv = rho <= cfg["tol"]
    assert conv[: cfg["b"]].all()
    AV = A @ Vg - Ug * Sg
    ATU = A.T @ Ug - Vg * Sg
    e1 = np.linalg.norm(AV, axis=0)
    e2 = np.linalg.norm(ATU, axis=0)
    # each computed value lies within its residuals of some exact one, and
    # below the i-th exact one (interlacing: U^T A V = Sigma is a compression)
    near = np.abs(Sg[:, None] - sig[None, :2 * r + 50]).min(axis=1)
    assert np.all(near <= e1 + e2 + 1e-13 * sig[0])
    assert np.all(Sg <= sig[:r] * (1 + 1e-12))
    assert np.abs(Sg - sig[:r])[conv].max() / sig[0] <= 1e-10
    assert np.abs(rho - e1 / sig[0]).max() <= 1e-12
    assert np.abs(Ug.T @ Ug - np.eye(r)).max() <= 1e-12
    assert np.abs(Vg.T @ Vg - np.eye(r)).max() <= 1e-12


def test_c4_rsvd_properties(c4):
    cfg, A, Ad, sig = c4
    r = cfg["r"]
    with T.TruncatedSVD(Ad) as h:
        h.set_seed(SEEDS["C4"])
        h.rsvd(r, cfg["rsvd_p"], cfg["rsvd_q"])
        Ug, Sg, Vg = h.get()
    assert np.abs(Ug.T @ Ug - np.eye(r)).max() <= 1e-12
    assert np.abs(Vg.T @ Vg - np.eye(r)).max() <= 1e-12
    f = np.linalg.norm(A.T @ Ug - Vg * Sg, axis=0) / sig[0]
    assert f.max() <= 1e-11
    e1 = np.linalg.norm(A @ Vg - Ug * Sg, axis=0)
    # Rayleigh-Ritz values from a subspace lie below the exact ones (Cauchy
    # interlacing for U^T A V = Sigma) and within Weyl's bound of them
    assert np.all(Sg <= sig[:r] * (1 + 1e-12))
    near = np.abs(Sg[:, None] - sig[None, :]).min(axis=1)
    assert np.all(near <= e1 + f * sig[0] + 1e-13 * sig[0])
