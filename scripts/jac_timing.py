"""Per-phase cycle counts of the register Jacobi (CTA 0), from an A/B build
compiled with -DJAC_TIMING (TSVD_LIB=ab_libs/libtsvd_jt.so)."""
import ctypes as C
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402

L = T.lib()
B = torch.from_numpy(np.load(os.path.join(os.path.dirname(__file__), "B384_lanczos.npy"))).cuda()
d = B.shape[0]
Ub = torch.empty((d, d), dtype=torch.float64, device="cuda")
Vb = torch.empty_like(Ub)
S = torch.empty(d, dtype=torch.float64, device="cuda")
T.dbg_small_svd(B, Ub, S, Vb)
torch.cuda.synchronize()
L.tsvd_dev_jacobi_timing_reset()
sw = T.dbg_small_svd(B, Ub, S, Vb)
torch.cuda.synchronize()
out = (C.c_ulonglong * 8)()
L.tsvd_dev_jacobi_timing(out)
v = list(out)
rounds = v[4]
names = ["wait+sync", "loads", "inner steps", "store+fence+publish", "rounds", "loop top"]
tot = sum(v[k] for k in (0, 1, 2, 3, 5))
print(f"sweeps {sw} rounds {rounds} total cycles {tot} ({tot / 1.9e3:.0f} us at 1.9 GHz)")
for k in (0, 1, 2, 3, 5):
    print(f"  {names[k]:22s} {v[k] / max(1, rounds):9.0f} cycles/round  {100 * v[k] / tot:5.1f}%")
