"""Full-size parity against the oracle itself (-m gpu, slow): the library's
solve and oracle/ (numpy/scipy fp64, Alg. 2 / Alg. 1 step by step) run on
the SAME bytes of BASELINE.json's configs, in the launch configuration
bench.py times (device-resident A, the bench's seeds and parameters).

North_star tolerances over triplets converged in both runs:
  |s_i - s_i^oracle| / s_1 <= 1e-10,  ||A v_i - s_i u_i|| / s_1 <= 1e-8,
  ||U^T U - I||_max, ||V^T V - I||_max <= 1e-12,
and the singular vectors, after sign alignment (reading R28), within the
Davis-Kahan bound of their residuals: a converged pair (u_i, v_i) with
residual e_i s_1 lies within angle ~ e_i s_1 / gap_i of the exact one
(A^T u_i = s_i v_i holds to rounding for Alg. 2's outputs, A^T Pbar_k =
P_k B_k^T, reading R1), so two converged runs differ by at most
(e_i + e_i^oracle) s_1 / gap_i (factor 4 margin).  These tests catch a
converged but WRONG triplet (a missed sigma in the top r), which residual
and orthogonality checks alone cannot.

Host cost on the GPU box (16 threads): C2 oracle ~40 s, C4 ~15 s, C3 RandSVD
q = 2 ~80 s.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import oracle  # noqa: E402
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import CONFIGS, SEEDS, dense_prescribed, powerlaw_csr, spectrum_eq16  # noqa: E402


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gaps(S):
    """Distance of each sigma_i to its nearest neighbour in S."""
    d = np.abs(np.diff(S))
    return np.minimum(np.r_[np.inf, d], np.r_[d, np.inf])


def _compare(op, Ug, Sg, Vg, conv_g, ro, conv_o, sig_next):
    """North_star tolerances + vector parity on triplets converged in both."""
    r = len(Sg)
    both = conv_g & conv_o
    assert both.sum() > 0
    s1 = ro.S[0]
    assert np.abs(Sg - ro.S)[both].max() / s1 <= 1e-10
    eg, _ = oracle.residuals(op, Ug, Sg, Vg)
    eo, _ = oracle.residuals(op, ro.U, ro.S, ro.V)
    assert eg[conv_g].max() <= 1e-8
    assert np.abs(Ug.T @ Ug - np.eye(r)).max() <= 1e-12
    assert np.abs(Vg.T @ Vg - np.eye(r)).max() <= 1e-12
    # gaps: to the neighbours inside the top r and to sigma_{r+1} (oracle's
    # estimate of the next value bounds the last gap from below)
    g = _gaps(np.r_[ro.S, sig_next])[:r]
    for i in np.where(both)[0]:
        bound = 4.0 * (eg[i] + eo[i]) * s1 / g[i] + 1e-12
        for Xg, Xo in ((Ug, ro.U), (Vg, ro.V)):
            sgn = np.sign(Xg[:, i] @ Xo[:, i])
            assert np.abs(sgn * Xg[:, i] - Xo[:, i]).max() <= bound, (i, bound)
    return eg, eo


def _lanczos_pair(cfg, seed, host_A, dev_A):
    """GPU solve (bench call sequence) and oracle solve on the same bytes."""
    m, n, r, b, d = cfg["m"], cfg["n"], cfg["r"], cfg["b"], cfg["d"]
    kw = dict(csr=dev_A, shape=(m, n)) if isinstance(dev_A, tuple) else dict(A=dev_A)
    with T.TruncatedSVD(**kw) as h:
        h.set_seed(seed)
        st = h.block_lanczos(r, b, cfg["tol"], cfg["maxit"], d=d)
        Ug, Sg, Vg = h.get()
        rho_g = h.rho()
        info = h.info()
    op = oracle.Operator(csr=host_A, shape=(m, n)) if isinstance(host_A, tuple) \
        else oracle.Operator(dense=host_A)
    ro = oracle.lancsvd(op, r, b, d, cfg["tol"], cfg["maxit"], seed, debug=True)
    return op, st, info, Ug, Sg, Vg, rho_g, ro


def test_c2_lanczos_vs_oracle():
    """C2 (m = n = 1e6, nnz 9.9e6, r = 50, b = 16, d = 384): the bench's
    default workload, solved by the library and by the oracle."""
    _cuda()
    cfg = CONFIGS["C2"]
    csr = powerlaw_csr(cfg["m"], cfg["n"], cfg["nnz"], cfg["alpha"], SEEDS["C2"])
    dev = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in csr)
    op, st, info, Ug, Sg, Vg, rho_g, ro = _lanczos_pair(cfg, SEEDS["C2"], csr, dev)
    assert st == T.TSVD_OK and ro.converged
    assert info["cycles"] == ro.cycles
    conv_g = rho_g <= cfg["tol"]
    conv_o = ro.rho <= cfg["tol"] * ro.S[0]
    assert conv_g.all() and conv_o.all()
    S_all = ro.debug["S_all"]
    _compare(op, Ug, Sg, Vg, conv_g, ro, conv_o, S_all[cfg["r"]])


def test_c4_lanczos_vs_oracle():
    """C4 (dense 40000 x 20000, Eq. 16 spectrum, r = 200, b = 32, d = 704)."""
    _cuda()
    cfg = CONFIGS["C4"]
    sig = spectrum_eq16(cfg["n"])
    A = dense_prescribed(cfg["m"], cfg["n"], sig, SEEDS["C4"], n_reflectors=4)
    op, st, info, Ug, Sg, Vg, rho_g, ro = _lanczos_pair(cfg, SEEDS["C4"], A,
                                                        torch.from_numpy(A).cuda())
    assert st in (T.TSVD_OK, T.TSVD_WARN_NOTCONV)
    assert info["cycles"] == ro.cycles
    conv_g = rho_g <= cfg["tol"]
    conv_o = ro.rho <= cfg["tol"] * ro.S[0]
    assert (conv_g == conv_o).all()
    eg, eo = _compare(op, Ug, Sg, Vg, conv_g, ro, conv_o, np.sort(sig)[::-1][cfg["r"]])
    # both also sit on the prescribed spectrum (closed form)
    exact = np.sort(sig)[::-1][: cfg["r"]]
    assert np.abs(Sg - exact)[conv_g].max() / exact[0] <= 1e-10


def test_c3_rsvd_vs_oracle():
    """C3 RandSVD q = 2 (r = 100, p = 10): at finite q the result is defined
    by the iteration (Alg. 1), so it is compared with the
    oracle's iterate from the same Philox start and the same CGS-QR panels:
    sigma to 1e-10 sigma_1, and the Ritz vectors whose Ritz values are
    separated (relative gap > 1e-3) to 1e-8."""
    _cuda()
    cfg = CONFIGS["C3"]
    m, n, r, p, q = cfg["m"], cfg["n"], cfg["r"], cfg["rsvd_p"], cfg["rsvd_q"]
    csr = powerlaw_csr(m, n, cfg["nnz"], cfg["alpha"], SEEDS["C3"])
    dev = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in csr)
    with T.TruncatedSVD(csr=dev, shape=(m, n)) as h:
        h.set_seed(SEEDS["C3"])
        h.rsvd(r, p, q)
        Ug, Sg, Vg = h.get()
    op = oracle.Operator(csr=csr, shape=(m, n))
    ro = oracle.randsvd(op, r=r, p=p, q=q, b_qr=16, seed=SEEDS["C3"])
    assert np.abs(Sg - ro.S).max() / ro.S[0] <= 1e-10
    g = _gaps(ro.S) / ro.S[0]
    sep = g > 1e-3
    assert sep.sum() > 0
    for Xg, Xo in ((Ug, ro.U), (Vg, ro.V)):
        sgn = np.sign(np.einsum("ij,ij->j", Xg, Xo))
        assert np.abs(Xg * sgn - Xo)[:, sep].max() <= 1e-8
    eg, _ = oracle.residuals(op, Ug, Sg, Vg)
    eo, _ = oracle.residuals(op, ro.U, ro.S, ro.V)
    assert np.abs(eg - eo).max() <= 1e-8
