"""Input generators (tsvd_inputs/, no method arithmetic): the device G1
generator used for C5 follows the same recipe as the host one (SURVEY 8(d):
Chung-Lu, Pareto alpha = 2.5 row lengths and column weights, duplicates
summed, N(0,1) values).  Run on the CPU device here."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from tsvd_inputs import powerlaw_csr, powerlaw_csr_device  # noqa: E402


def _canonical(rp, ci, m, n):
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == len(ci)
    assert ci.min() >= 0 and ci.max() < n
    # strictly increasing column indices inside every row (sorted, no duplicates)
    d = np.diff(ci.astype(np.int64))
    starts = rp[1:-1]
    inner = np.ones(len(ci) - 1, bool)
    inner[starts[(starts > 0) & (starts < len(ci))] - 1] = False
    assert np.all(d[inner] > 0)


def test_device_generator_recipe():
    m, n, nnz = 200_000, 150_000, 2_000_000
    rp, ci, va = (x.numpy() for x in powerlaw_csr_device(m, n, nnz, 2.5, seed=5, device="cpu"))
    _canonical(rp, ci, m, n)
    assert abs(len(ci) - nnz) <= 0.01 * nnz                      # within 1% after dedup
    rp2, ci2, va2 = powerlaw_csr(m, n, nnz, 2.5, seed=5)
    L, L2 = np.diff(rp), np.diff(rp2)
    # same row-length law: mean, tail quantiles and max within sampling noise
    assert abs(L.mean() - L2.mean()) <= 0.02 * L2.mean()
    for q in (50, 90, 99):
        assert abs(np.percentile(L, q) - np.percentile(L2, q)) <= 0.1 * np.percentile(L2, q) + 1
    c, c2 = np.bincount(ci, minlength=n), np.bincount(ci2, minlength=n)
    for q in (50, 90, 99):
        assert abs(np.percentile(c, q) - np.percentile(c2, q)) <= 0.1 * np.percentile(c2, q) + 1
    # values: N(0,1) (sums of duplicates are rare)
    assert abs(va.mean()) < 0.01 and abs(va.std() - 1.0) < 0.02


def test_device_generator_deterministic():
    a = powerlaw_csr_device(5000, 4000, 40000, 2.5, seed=9, device="cpu")
    b = powerlaw_csr_device(5000, 4000, 40000, 2.5, seed=9, device="cpu")
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_blockdiag_device_g2_closed_form_spectrum():
    """G2 at C5 scale is built by blockdiag_csr_device (torch); on the CPU at
    a small size its dense SVD equals the prescribed spectrum (Householder
    reflector blocks: sigma(B_t) = s_t exactly) and the CSR is canonical."""
    torch = pytest.importorskip("torch")
    import scipy.sparse as sp
    from tsvd_inputs import blockdiag_csr_device
    m = 2500
    rp, ci, va, sig = blockdiag_csr_device(m, m, 3.0, 2.5, 5, np.linspace(50, 30, 10),
                                           tail_max=5.0, device="cpu", chunk_rows=600)
    rp, ci, va = rp.numpy(), ci.numpy(), va.numpy()
    A = sp.csr_matrix((va, ci.astype(np.int64), rp), shape=(m, m))
    sv = np.linalg.svd(A.toarray(), compute_uv=False)
    assert np.abs(sv - sig).max() <= 1e-13 * sig[0]
    assert np.allclose(sig[:10], np.linspace(50, 30, 10)) and sig[10] <= 5.0
    assert all(np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0) for i in range(m))
