"""One launch of a hot kernel at a KNOWN shape, for the ncu DRAM-traffic
capture (roofline.traffic in bench.py).  Development tool, not the bench.

    ncu --set full -k regex:<kernel> -c 1 python scripts/traffic_probe.py nn|tn|spmm|dense_nn|dense_tn

Prints the launch's algorithmic bytes so that
scripts/summarize_ncu.py can form dram_bytes / algorithmic_bytes.
  nn       CGS-CQR2 pass B shape on C2's m side: Z = Y - P H, q = 1e6, s = 304, w = 16
  tn       CGS-CQR2 pass A: H = P^T Y at the same shape
  spmm     C2's A.X (CSR, w = 16)
  dense_nn C4's A.X (dense 40000 x 20000, w = 32)
  dense_tn C4's A^T.X
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402


def main(mode):
    T.lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    if mode in ("nn", "tn"):
        q, s, w = 1_000_000, 304, 16
        X = torch.randn((q, s + w), dtype=torch.float64, device="cuda", generator=g)
        if mode == "nn":
            H = torch.randn((s, w), dtype=torch.float64, device="cuda", generator=g)
            Z = X[:, s:]
            T.dbg_gemm_nn(X[:, :s], H, Z, -1.0, 1.0)
            alg = 8.0 * q * (s + 2 * w)
        else:
            C = torch.empty((s, w), dtype=torch.float64, device="cuda")
            T.dbg_gemm_tn(X[:, :s], X[:, s:], C)
            alg = 8.0 * q * (s + w)
        shape = dict(q=q, s=s, w=w)
    elif mode == "spmm":
        from tsvd_inputs import CONFIGS, SEEDS, powerlaw_csr
        cfg = CONFIGS["C2"]
        m, n, w = cfg["m"], cfg["n"], 16
        rp, ci, va = powerlaw_csr(m, n, cfg["nnz"], cfg["alpha"], SEEDS["C2"])
        dev = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (rp, ci, va))
        h = T.TruncatedSVD(csr=dev, shape=(m, n))
        X = torch.randn((n, w), dtype=torch.float64, device="cuda", generator=g)
        Y = torch.empty((m, w), dtype=torch.float64, device="cuda")
        T.dbg_apply(h, False, X, Y)
        nnz = len(ci)
        alg = 12.0 * nnz + 8.0 * (m + 1) + 8.0 * w * (m + n)
        shape = dict(m=m, n=n, nnz=nnz, w=w)
    else:
        m, n, w = 40_000, 20_000, 32
        A = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
        h = T.TruncatedSVD(A)
        if mode == "dense_nn":
            X = torch.randn((n, w), dtype=torch.float64, device="cuda", generator=g)
            Y = torch.empty((m, w), dtype=torch.float64, device="cuda")
            T.dbg_apply(h, False, X, Y)
        else:
            X = torch.randn((m, w), dtype=torch.float64, device="cuda", generator=g)
            Y = torch.empty((n, w), dtype=torch.float64, device="cuda")
            T.dbg_apply(h, True, X, Y)
        alg = 8.0 * (m * n + w * (m + n))
        shape = dict(m=m, n=n, w=w, flops=2.0 * m * n * w)
    torch.cuda.synchronize()
    print(json.dumps(dict(mode=mode, alg_bytes=alg, **shape)))


if __name__ == "__main__":
    main(sys.argv[1])
