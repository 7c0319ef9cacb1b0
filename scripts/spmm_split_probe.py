"""Probe: does cutting A's columns into K ranges (so the gathered X slice
fits in L2) speed up the C2 SpMM?  Times A_k . X_k for each column range k
as separate handles (no accumulation) against the whole product.
Development tool (gpurun), not part of the bench."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402
from scripts.bench_kernels import timeit  # noqa: E402
from tsvd_inputs import powerlaw_csr  # noqa: E402

m = n = 1_000_000
w, d = 16, 384
rp, ci, va = powerlaw_csr(m, n, 10_000_000, 2.5, seed=0x2403062182)
P = torch.randn((n, d), dtype=torch.float64, device="cuda")
Pb = torch.randn((m, d + w), dtype=torch.float64, device="cuda")
X, Y = P[:, 64:64 + w], Pb[:, 64:64 + w]
h = T.TruncatedSVD(csr=(rp, ci, va), shape=(m, n))
full = timeit(lambda: T.dbg_apply(h, False, X, Y), reps=10, warm=3)
print(f"full: {full:.4f} ms", flush=True)
h.close()
# per-call floor (launch + the entry point's stream synchronisation)
ht = T.TruncatedSVD(csr=(np.arange(1001, dtype=np.int64), np.arange(1000, dtype=np.int32),
                         np.ones(1000)), shape=(1000, 1000))
floor = timeit(lambda: T.dbg_apply(ht, False, X[:1000], Y[:1000]), reps=10, warm=3)
ht.close()
print(f"per-call floor: {floor:.4f} ms", flush=True)
rows = np.repeat(np.arange(m), np.diff(rp))
for K in (2, 3, 4, 8):
    hs, Xs = [], []
    for k in range(K):
        c0, c1 = k * n // K, (k + 1) * n // K
        sel = (ci >= c0) & (ci < c1)
        r = rows[sel]
        rpk = np.zeros(m + 1, dtype=np.int64)
        np.add.at(rpk, r + 1, 1)
        rpk = np.cumsum(rpk)
        hs.append(T.TruncatedSVD(csr=(rpk, (ci[sel] - c0).astype(np.int32), va[sel]),
                                 shape=(m, c1 - c0)))
        Xs.append(X[c0:c1])
    ts = [timeit(lambda: T.dbg_apply(hs[k], False, Xs[k], Y), reps=10, warm=3) for k in range(K)]
    print(f"K={K}: parts {' '.join(f'{t:.4f}' for t in ts)} sum {sum(ts):.4f} ms "
          f"(full {full:.4f})", flush=True)
    for hh in hs:
        hh.close()
