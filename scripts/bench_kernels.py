"""Micro-benchmarks of single building blocks through the tsvd_dbg_* entry
points (CUDA-event timed, after warm-up).  Development tool, not the bench.

    python scripts/bench_kernels.py [svd] [tn] [nn] [spmm] [cqr]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402

HBM = 6548.5


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def svd_bench():
    for d in [int(x) for x in os.environ.get("SVD_D", "28,128,200,384,450,704").split(",")]:
        rng = np.random.default_rng(d)
        B = torch.from_numpy(np.tril(rng.standard_normal((d, d))) * (0.97 ** np.arange(d))).cuda()
        if os.environ.get("SVD_LANCZOS") and d != 384:
            # Lanczos-shaped lower block-bidiagonal B (b = 32), as tests/test_gpu_kernels.py
            bb, B0 = 32, np.zeros((d, d))
            for i in range(d // bb):
                sc = 100.0 * 0.97 ** i
                B0[i * bb:(i + 1) * bb, i * bb:(i + 1) * bb] = sc * np.tril(rng.standard_normal((bb, bb)))
                if (i + 2) * bb <= d:
                    B0[(i + 1) * bb:(i + 2) * bb, i * bb:(i + 1) * bb] = 0.3 * sc * np.triu(
                        rng.standard_normal((bb, bb)))
            B = torch.from_numpy(B0).cuda()
        if d == 384 and os.path.exists(os.path.join(os.path.dirname(__file__), "B384_lanczos.npy")):
            B = torch.from_numpy(np.load(os.path.join(os.path.dirname(__file__), "B384_lanczos.npy"))).cuda()
        Ub = torch.empty((d, d), dtype=torch.float64, device="cuda")
        Vb = torch.empty_like(Ub)
        S = torch.empty(d, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: T.dbg_small_svd(B, Ub, S, Vb), reps=3, warm=1)
        sweeps = T.dbg_small_svd(B, Ub, S, Vb)
        Bn = B.cpu().numpy()
        sv = np.linalg.svd(Bn, compute_uv=False)
        err = np.abs(S.cpu().numpy() - sv).max() / sv[0]
        Vn, Un, Sn = Vb.cpu().numpy(), Ub.cpu().numpy(), S.cpu().numpy()
        orth = np.abs(Vn.T @ Vn - np.eye(d)).max()
        rec = np.abs(Un @ np.diag(Sn) @ Vn.T - Bn).max() / sv[0]
        print(f"small_svd d={d}: {ms:.3f} ms  sweeps {sweeps}  sigma err {err:.1e}  "
              f"V orth {orth:.1e}  recon {rec:.1e}", flush=True)


def tn_bench():
    for q, s, w in ((1_000_000, 384, 16), (1_000_000, 128, 16), (1_000_000, 16, 16),
                    (1_000_000, 704, 32), (1_000_000, 384, 32)):
        X = torch.randn((q, s + w), dtype=torch.float64, device="cuda")
        C = torch.empty((s, w), dtype=torch.float64, device="cuda")
        Xv, Yv = X[:, :s], X[:, s:]
        ms = timeit(lambda: T.lib().tsvd_dbg_gemm_tn(Xv.data_ptr(), X.stride(0), Yv.data_ptr(),
                                                     X.stride(0), q, s, w, C.data_ptr(), None))
        gb = 8.0 * q * (s + w) / (ms * 1e-3) / 1e9
        tf = 2.0 * q * s * w / (ms * 1e-3) / 1e12
        print(f"gemm_tn q={q} s={s} w={w}: {ms:.3f} ms  {gb:.0f} GB/s ({gb / HBM:.2f} of HBM) "
              f"{tf:.1f} TF/s ({tf / 37.1:.2f} of DMMA)", flush=True)


def nn_bench():
    for q, s, w in ((1_000_000, 384, 16), (1_000_000, 128, 16), (1_000_000, 0, 16),
                    (1_000_000, 704, 32), (1_000_000, 384, 32), (4_000_000, 0, 32)):
        X = torch.randn((q, max(s, 1) + w), dtype=torch.float64, device="cuda")
        H = torch.randn((max(s, 1), w), dtype=torch.float64, device="cuda")
        Z = torch.empty((q, w), dtype=torch.float64, device="cuda")
        Y = X[:, max(s, 1):]
        ms = timeit(lambda: T.lib().tsvd_dbg_gemm_nn(X.data_ptr(), X.stride(0), H.data_ptr(), w,
                                                     Z.data_ptr(), w, q, s, w, -1.0, 1.0, None))
        gb = 8.0 * q * (s + 2 * w) / (ms * 1e-3) / 1e9
        tf = 2.0 * q * (s + w) * w / (ms * 1e-3) / 1e12
        print(f"gemm_nn q={q} s={s} w={w}: {ms:.3f} ms  {gb:.0f} GB/s ({gb / HBM:.2f} of HBM) "
              f"{tf:.1f} TF/s ({tf / 37.1:.2f} of DMMA)", flush=True)


def nn32_bench():
    """the w = 32 NN pass at C3's largest s (the dominant kernel of C3 / C5)
    and the TN pass beside it, for ncu"""
    q, s, w = 1_000_000, 640, 32
    X = torch.randn((q, s + w), dtype=torch.float64, device="cuda")
    H = torch.randn((s, w), dtype=torch.float64, device="cuda")
    Z = torch.empty((q, w), dtype=torch.float64, device="cuda")
    C = torch.empty((s, w), dtype=torch.float64, device="cuda")
    G = torch.empty((148, w, w), dtype=torch.float64, device="cuda")
    L = T.lib()
    ms = timeit(lambda: L.tsvd_dbg_gemm_nn(X.data_ptr(), s + w, H.data_ptr(), w, Z.data_ptr(), w,
                                           q, s, w, -1.0, 1.0, None))
    tf = 2.0 * q * (s + w) * w / (ms * 1e-3) / 1e12
    print(f"gemm_nn q={q} s={s} w={w}: {ms:.3f} ms  {tf:.1f} TF/s ({tf / 37.1:.2f} of DMMA)",
          flush=True)
    ms = timeit(lambda: L.tsvd_dbg_gemm_tn(X.data_ptr(), s + w, X[:, s:].data_ptr(), s + w, q, s,
                                           w, C.data_ptr(), None))
    tf = 2.0 * q * s * w / (ms * 1e-3) / 1e12
    print(f"gemm_tn q={q} s={s} w={w}: {ms:.3f} ms  {tf:.1f} TF/s ({tf / 37.1:.2f} of DMMA)",
          flush=True)


def sweep_bench():
    q, w = 1_000_000, 16
    X = torch.randn((q, 400), dtype=torch.float64, device="cuda")
    H = torch.randn((400, w), dtype=torch.float64, device="cuda")
    Z = torch.empty((q, w), dtype=torch.float64, device="cuda")
    C = torch.empty((400, w), dtype=torch.float64, device="cuda")
    L = T.lib()
    for s in (16, 32, 64, 96, 128, 192, 256, 320, 384):
        Y = X[:, s:]
        ms_tn = timeit(lambda: L.tsvd_dbg_gemm_tn(X.data_ptr(), 400, Y.data_ptr(), 400, q, s, w,
                                                  C.data_ptr(), None))
        ms_nn = timeit(lambda: L.tsvd_dbg_gemm_nn(X.data_ptr(), 400, H.data_ptr(), w, Z.data_ptr(),
                                                  w, q, s, w, -1.0, 1.0, None))
        gtn = 8.0 * q * (s + w) / (ms_tn * 1e-3) / 1e9
        gnn = 8.0 * q * (s + 2 * w) / (ms_nn * 1e-3) / 1e9
        print(f"s={s:4d}  tn {ms_tn:.3f} ms {gtn:5.0f} GB/s ({gtn / HBM:.2f})   "
              f"nn {ms_nn:.3f} ms {gnn:5.0f} GB/s ({gnn / HBM:.2f})", flush=True)


def out_bench():
    """output products Z = X H (beta = 0), w = r = 50 and 64 (U = Pbar Ubar_r)"""
    q, s = 1_000_000, 384
    X = torch.randn((q, s + 16), dtype=torch.float64, device="cuda")
    H = torch.randn((s, s), dtype=torch.float64, device="cuda")
    for w in (50, 64, 16):
        Z = torch.empty((q, w), dtype=torch.float64, device="cuda")
        ms = timeit(lambda: T.lib().tsvd_dbg_gemm_nn(X.data_ptr(), X.stride(0), H.data_ptr(), s,
                                                     Z.data_ptr(), w, q, s, w, 1.0, 0.0, None))
        tf = 2.0 * q * s * w / (ms * 1e-3) / 1e12
        gb = 8.0 * q * (s + w) / (ms * 1e-3) / 1e9
        print(f"gemm_nn(out) q={q} s={s} w={w}: {ms:.3f} ms  {tf:.1f} TF/s  {gb:.0f} GB/s", flush=True)


def nn0_bench():
    """single s=0 and s=384 gemm_nn launches (for ncu)"""
    q, w = 1_000_000, 16
    X = torch.randn((q, 400), dtype=torch.float64, device="cuda")
    H = torch.randn((400, w), dtype=torch.float64, device="cuda")
    Z = torch.randn((q, w), dtype=torch.float64, device="cuda")
    Tm = torch.triu(torch.randn((w, w), dtype=torch.float64, device="cuda"))
    G = torch.empty((148 * 2, w, w), dtype=torch.float64, device="cuda")
    L = T.lib()
    for s in (0, 384):
        L.tsvd_dbg_gemm_nn(X.data_ptr(), 400, H.data_ptr(), w, Z.data_ptr(), w, q, s, w, -1.0, 1.0, None)
    torch.cuda.synchronize()


def spmm_bench():
    """SpMM on the solver's operand layout: X and Y are column slices of the
    row-major bases (ld = d + b on the m side, d on the n side)."""
    from tsvd_inputs import powerlaw_csr
    shapes = os.environ.get("SPMM_CFG", "C2,C3").split(",")
    for cfgn in shapes:
        if cfgn == "C2":
            m, n, nnz, w, d = 1_000_000, 1_000_000, 10_000_000, 16, 384
            seed = 0x2403062182
        else:
            m, n, nnz, w, d = 4_000_000, 500_000, 50_000_000, 32, 640
            seed = 0x2403062183
        csr = powerlaw_csr(m, n, nnz, 2.5, seed=seed)
        h = T.TruncatedSVD(csr=csr, shape=(m, n))
        nnz = len(csr[1])
        Pb = torch.randn((m, d + w), dtype=torch.float64, device="cuda")
        P = torch.randn((n, d), dtype=torch.float64, device="cuda")
        for tr in (False, True):
            # A.Q: X = n-side slice of P, Y = m-side slice of Pbar; A^T.Qbar the reverse
            X, Y = (Pb[:, 64:64 + w], P[:, 64:64 + w]) if tr else (P[:, 64:64 + w], Pb[:, 64:64 + w])
            ms = timeit(lambda: T.dbg_apply(h, tr, X, Y))
            rows, cols = (n, m) if tr else (m, n)
            gb = (12.0 * nnz + 8 * (rows + 1) + 8.0 * w * (rows + cols)) / (ms * 1e-3) / 1e9
            print(f"spmm {cfgn} w={w} trans={tr}: "
                  f"{ms:.3f} ms  {gb:.0f} GB/s compulsory ({gb / HBM:.2f} of HBM)", flush=True)
        h.close()
        del Pb, P


def dense_bench():
    """C4's dense products A.X / A^T.X (FP64 DMMA-bound for w >= 32)"""
    m, n = 40_000, 20_000
    A = torch.randn((m, n), dtype=torch.float64, device="cuda")
    h = T.TruncatedSVD(A)
    for w in (16, 32, 210):
        X = torch.randn((n, w), dtype=torch.float64, device="cuda")
        Xt = torch.randn((m, w), dtype=torch.float64, device="cuda")
        Y = torch.empty((m, w), dtype=torch.float64, device="cuda")
        Z = torch.empty((n, w), dtype=torch.float64, device="cuda")
        for tr, xin, yout in ((False, X, Y), (True, Xt, Z)):
            ms = timeit(lambda: T.dbg_apply(h, tr, xin, yout))
            tf = 2.0 * m * n * w / (ms * 1e-3) / 1e12
            gb = 8.0 * (m * n + w * (m + n)) / (ms * 1e-3) / 1e9
            print(f"dense w={w} trans={tr}: {ms:.3f} ms  {tf:.1f} TF/s ({tf / 37.1:.2f} of DMMA)  "
                  f"{gb:.0f} GB/s ({gb / HBM:.2f} of HBM)", flush=True)
    h.close()


def cqr_bench():
    q = 1_000_000
    for s, w in ((0, 16), (192, 16), (384, 16), (640, 32)):
        basis = torch.randn((q, s + w), dtype=torch.float64, device="cuda")
        if s:
            Qp, _ = torch.linalg.qr(basis[:, :s])
            basis[:, :s] = Qp
        H = torch.empty((max(s, 1), w), dtype=torch.float64, device="cuda")
        R = torch.empty((w, w), dtype=torch.float64, device="cuda")
        Y0 = basis[:, s:].clone()

        def run():
            basis[:, s:] = Y0
            T.dbg_cgs_cqr2(basis, s, w, H, R)
        ms = timeit(run, reps=3, warm=1)
        print(f"cgs_cqr2 q={q} s={s} w={w}: {ms:.3f} ms (incl. copy)", flush=True)


if __name__ == "__main__":
    T.lib()
    what = sys.argv[1:] or ["svd", "tn", "nn", "spmm", "cqr"]
    for w in what:
        globals()[f"{w}_bench"]()
