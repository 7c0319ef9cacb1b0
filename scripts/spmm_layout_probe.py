"""Probe: does the gathered operand's layout matter for the C2 SpMM?  X as
a 16-column slice of the n x 384 basis (ld = 384: rows 128 B apart by 3 KB,
3 GB spanned) vs the same values contiguous (ld = 16: 128 MB spanned, far
fewer pages for the random row gathers).  Development tool (gpurun)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402
from scripts.bench_kernels import timeit  # noqa: E402
from tsvd_inputs import powerlaw_csr  # noqa: E402

m = n = 1_000_000
w, d = 16, 384
rp, ci, va = powerlaw_csr(m, n, 10_000_000, 2.5, seed=0x2403062182)
h = T.TruncatedSVD(csr=(rp, ci, va), shape=(m, n))
P = torch.randn((n, d), dtype=torch.float64, device="cuda")
Pb = torch.randn((m, d + w), dtype=torch.float64, device="cuda")
Xs, Ys = P[:, 64:64 + w], Pb[:, 64:64 + w]
Xc, Yc = Xs.contiguous(), torch.empty((m, w), dtype=torch.float64, device="cuda")
Xbs, Ybs = Pb[:, 64:64 + w], P[:, 64:64 + w]   # A^T: gather from the m side
Xbc = Xbs.contiguous()
Ytc = torch.empty((n, w), dtype=torch.float64, device="cuda")
for name, fn in [
        ("A.X   strided X, strided Y", lambda: T.dbg_apply(h, False, Xs, Ys)),
        ("A.X   contig  X, strided Y", lambda: T.dbg_apply(h, False, Xc, Ys)),
        ("A.X   contig  X, contig  Y", lambda: T.dbg_apply(h, False, Xc, Yc)),
        ("A^T.X strided X, strided Y", lambda: T.dbg_apply(h, True, Xbs, Ybs)),
        ("A^T.X contig  X, strided Y", lambda: T.dbg_apply(h, True, Xbc, Ybs)),
        ("A^T.X contig  X, contig  Y", lambda: T.dbg_apply(h, True, Xbc, Ytc)),
        ("copy of the X slice (torch)", lambda: Xc.copy_(Xs))]:
    print(f"{name}: {timeit(fn, reps=20, warm=3):.4f} ms", flush=True)
h.close()
