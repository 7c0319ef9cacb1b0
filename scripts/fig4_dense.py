"""the paper's dense workload at its own sizes on one B200
(Sec. 4.2, Fig. 4): A = X Sigma Y^T (Eq. 15) with n = 10 000,
m in {1e5, 2.5e5, 7.5e5, 1e6}, Sigma by Eq. 16 (set reading R14), 10 wanted
triplets, b = 16.  LancSVD with the paper's r = 64 (Krylov dimension d = 64,
reading R7) and p = 1 or 4 iterations (restart cycles); RandSVD with the
paper's r = 16 (l = 16: r = 10 wanted + oversampling 6, reading R6) and
p = 6 or 24 iterations (q = p - 1 power iterations).  Reports the CUDA-event
time of each solve (median of 3 after one warm-up) and the relative residuals
R_i = ||A v_i - sigma_i u_i|| / sigma_i, i = 1..10 (Eq. 14 as corrected,
reading R13), computed by torch on the device, plus |sigma_i - sigma_i^true|/sigma_1.
A is built on the device with 4 random Householder reflectors per side
(exact spectrum, tsvd_inputs.dense_prescribed(xp="torch")).

    python scripts/fig4_dense.py [m ...]   -> one JSON line per run
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import dense_prescribed, spectrum_eq16  # noqa: E402

N = 10_000
RUNS = [("lanczos", 1), ("lanczos", 4), ("rsvd", 6), ("rsvd", 24)]


def main():
    ms = [int(float(x)) for x in sys.argv[1:]] or [100_000, 250_000, 750_000, 1_000_000]
    sig = spectrum_eq16(N)
    T.lib()
    for m in ms:
        A = dense_prescribed(m, N, sig, seed=0x2403062186 + m, n_reflectors=4, xp="torch",
                             device="cuda")
        torch.cuda.synchronize()
        for algo, p in RUNS:
            h = T.TruncatedSVD(A)
            h.set_seed(0x24030621)
            st = torch.cuda.current_stream()

            def solve():
                if algo == "lanczos":
                    return h.block_lanczos(10, 16, 1e-15, p, d=64)
                return h.rsvd(10, 6, p - 1)
            solve()
            times = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                solve()
                e1.record(st)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            info = h.info()
            U, S, V = h.get(device=True)
            h.close()
            R = (torch.linalg.vector_norm(A @ V - U * S, dim=0) / S).cpu().numpy()
            S = S.cpu().numpy()
            out = {"m": m, "n": N, "algo": algo,
                   "paper_setting": (f"LancSVD r=64 (d), p={p} iterations" if algo == "lanczos"
                                     else f"RandSVD r=16 (l), p={p} iterations (q={p - 1})"),
                   "ms_median": round(statistics.median(times), 3),
                   "ms_all": [round(t, 3) for t in times], "cycles": info["cycles"],
                   "R": [float(f"{x:.3e}") for x in R],
                   "sigma_err_max": float(np.abs(S - sig[:10]).max() / sig[0]),
                   "UtU_minus_I": float((U.T @ U - torch.eye(10, dtype=U.dtype, device=U.device)).abs().max())}
            print(json.dumps(out), flush=True)
            del U, V
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
