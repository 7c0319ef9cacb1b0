"""Diagnose CholQR breakdowns (CGS2 fallbacks) on C3-shaped inputs.
    python scripts/c3_debug.py SCALE B D MAXIT"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import powerlaw_csr  # noqa: E402

sc, b, d, maxit = float(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
m, n = int(4e6 * sc), int(5e5 * sc)
csr = powerlaw_csr(m, n, int(5e7 * sc), 2.5, 0x2403062183)
dev = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in csr)
h = T.TruncatedSVD(csr=dev, shape=(m, n))
h.set_seed(0x2403062183)
h.set_krylov_dim(d)
h.set_profiling(True)
t = time.time()
st = h.block_lanczos(100, b, 1e-8, maxit)
inf = h.info()
prof = h.profile()
print(f"scale {sc} b {b} d {d}: status {st} {time.time()-t:.1f}s info "
      f"cycles={inf['cycles']} nconv={inf['nconv']} breakdowns={inf['breakdowns']} "
      f"rho_max={inf['rho_max']:.2e} other_calls={prof['other']['calls']} "
      f"other_ms={prof['other']['ms']:.0f}", flush=True)
