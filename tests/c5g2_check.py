"""C5 (iii) accuracy at full scale, run in a fresh process by
tests/test_gpu_fullsize_c5.py: the G2 twin of C5 -- block-diagonal CSR,
m = n = 5e7, nnz ~1e9, generated on the device with a CLOSED-FORM spectrum
(tsvd_inputs.blockdiag_csr_device: top 100 singular values linspace(200,
100), the rest <= 20) -- solved by LancSVD to tol = 1e-8 on one GPU with the
bases' d = 160, b = 32 and thick restart keeping 128 Ritz pairs (formed in
place: the m x 128 panels do not fit next to 141 GB of bases).

Checks (north_star tolerances, over the converged triplets):
  * |sigma_i - sigma_i^exact| / sigma_1 <= 1e-10 (closed form, no oracle run
    needed at this size);
  * e_i = ||A v_i - s_i u_i|| / s_1 <= 1e-8 from tsvd_residuals (the
    library's own A.X and column norms; parity with oracle.residuals is
    pinned at smaller sizes by test_residuals_parity);
  * rho_i (Eq. 10) agrees with e_i.
Prints one JSON line; exit code 0 iff every check passed.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import CONFIGS, SEEDS, blockdiag_csr_device  # noqa: E402


def main():
    cfg = CONFIGS["C5g2"]
    m, n, r = cfg["m"], cfg["n"], cfg["r"]
    hi, lo, k = cfg["top"]
    t0 = time.time()
    rp, ci, va, sig = blockdiag_csr_device(m, n, cfg["mean_block"], cfg["alpha"], SEEDS["C5g2"],
                                           np.linspace(hi, lo, k), tail_max=cfg["tail_max"])
    out = {"nnz": int(ci.numel()), "gen_s": round(time.time() - t0, 1)}
    t0 = time.time()
    h = T.TruncatedSVD(csr=(rp, ci, va), shape=(m, n))
    del rp, ci, va
    torch.cuda.empty_cache()
    T.trim_memory(0)
    out["create_s"] = round(time.time() - t0, 1)
    h.set_seed(SEEDS["C5g2"])
    h.set_thick_restart(cfg["keep"])
    t0 = time.time()
    st = h.block_lanczos(r, cfg["b"], cfg["tol"], cfg["maxit"], d=cfg["d"])
    torch.cuda.synchronize()
    out["solve_s"] = round(time.time() - t0, 2)
    info = h.info()
    out["status"], out["info"] = st, {k2: info[k2] for k2 in
                                      ("cycles", "nconv", "breakdowns", "rho_max", "ms_total")}
    S = h.singular_values()
    rho = h.rho()
    e, _ = h.residuals()
    conv = rho <= cfg["tol"]
    exact = sig[:r]
    out["sigma_err"] = float(np.abs(S - exact)[conv].max() / exact[0]) if conv.any() else None
    out["e_max_conv"] = float(e[conv].max()) if conv.any() else None
    out["rho_vs_e"] = float(np.abs(rho - e).max())
    out["ok"] = bool(st == T.TSVD_OK and conv.all() and out["sigma_err"] <= 1e-10
                     and out["e_max_conv"] <= 1e-8 and out["rho_vs_e"] <= 1e-12)
    h.close()
    print(json.dumps(out), flush=True)
    return 0 if out["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
