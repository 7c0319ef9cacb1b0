"""C5 full-size checks, run in a fresh process by tests/test_gpu_fullsize_c5.py
(the solve needs ~178 GB of the device, so nothing else may hold memory).

  1. SpMM at C5 scale in the launch configuration of the solver (w = 32):
     sampled rows of A.X and of A^T.X recomputed on the host in fp64 from the
     CSR rows / columns, within the forward-error bound 2(K+1)u sum|a||x|.
  2. One fixed-work LancSVD cycle (r = 100, b = 32, d = 160, outputs in
     place): no breakdown, sigma descending and positive, rho finite, and the
     returned U / V columns orthonormal on sampled rows (U^T U over all rows
     is computed on the device by torch, independently of the library).
Prints one JSON line; exit code 0 iff every check passed.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import CONFIGS, SEEDS, powerlaw_csr_device  # noqa: E402

U = 2.0 ** -53


def main():
    cfg = CONFIGS["C5"]
    m, n = cfg["m"], cfg["n"]
    rp, ci, va = powerlaw_csr_device(m, n, cfg["nnz"], cfg["alpha"], SEEDS["C5"])
    h = T.TruncatedSVD(csr=(rp, ci, va), shape=(m, n))
    out = {"nnz": int(ci.numel())}
    g = torch.Generator(device="cuda").manual_seed(3)
    w = 32
    X = torch.randn((n, w), dtype=torch.float64, device="cuda", generator=g)
    Y = torch.full((m, w), float("nan"), dtype=torch.float64, device="cuda")
    T.dbg_apply(h, False, X, Y)
    rng = np.random.default_rng(0)
    lens = torch.diff(rp)
    rows = np.unique(np.concatenate([rng.integers(0, m, 200),
                                     torch.topk(lens, 8).indices.cpu().numpy()]))
    worst = 0.0
    for i in rows:
        b, e = int(rp[i]), int(rp[i + 1])
        cols = ci[b:e].long()
        vals = va[b:e].cpu().numpy()
        Xc = X[cols].cpu().numpy()
        ref = vals @ Xc
        bound = 2 * (len(vals) + 1) * U * (np.abs(vals) @ np.abs(Xc)) + 1e-300
        worst = max(worst, float(np.max(np.abs(Y[i].cpu().numpy() - ref) / bound)))
    out["spmm_rows_checked"] = int(len(rows))
    out["spmm_worst_over_bound"] = worst
    del Y
    # A^T.X: output row j = column j of A, gathered on the device by a compare
    Z = torch.full((n, w), float("nan"), dtype=torch.float64, device="cuda")
    Xt = X.new_empty((m, w)).normal_(generator=g)
    del X
    T.dbg_apply(h, True, Xt, Z)
    colcnt = torch.bincount(ci, minlength=n)
    cols_s = np.unique(np.concatenate([rng.integers(0, n, 16),
                                       torch.topk(colcnt, 4).indices.cpu().numpy()]))
    worst_t = 0.0
    for j in cols_s:
        pos = torch.nonzero(ci == int(j)).flatten()
        rr = torch.searchsorted(rp, pos, right=True) - 1
        vv = va[pos].cpu().numpy()
        Xr = Xt[rr].cpu().numpy()
        ref = vv @ Xr
        bound = 2 * (len(vv) + 1) * U * (np.abs(vv) @ np.abs(Xr)) + 1e-300
        worst_t = max(worst_t, float(np.max(np.abs(Z[int(j)].cpu().numpy() - ref) / bound)))
    out["spmm_t_cols_checked"] = int(len(cols_s))
    out["spmm_t_worst_over_bound"] = worst_t
    del Z, Xt, rp, ci, va, lens, colcnt
    torch.cuda.empty_cache()
    T.trim_memory(0)
    # one fixed-work cycle, outputs in place (AUTO)
    h.set_seed(SEEDS["C5"])
    h.set_krylov_dim(cfg["d"])
    st = h.block_lanczos(cfg["r"], cfg["b"], cfg["tol"], 1)
    info = h.info()
    out["status"] = int(st)
    out["info"] = {k: info[k] for k in ("cycles", "breakdowns", "replaced", "rho_max", "sigma1")}
    r = cfg["r"]
    S = np.empty(r)
    T._check(T.lib().tsvd_get(h._h, None, r, S.ctypes.data, None, r, T.TSVD_HOST), "tsvd_get")
    out["sigma_desc"] = bool(np.all(np.diff(S) <= 0) and S[-1] > 0)
    out["sigma1_matches_info"] = bool(S[0] == info["sigma1"])
    ok = (worst <= 1.0 and worst_t <= 1.0 and st in (T.TSVD_OK, T.TSVD_WARN_NOTCONV)
          and info["breakdowns"] == 0 and np.isfinite(info["rho_max"]) and out["sigma_desc"]
          and out["sigma1_matches_info"])
    out["ok"] = bool(ok)
    print(json.dumps(out), flush=True)
    h.close()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
