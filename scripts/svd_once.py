"""One small_svd call at dimension d (for ncu)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T
d = int(sys.argv[1]) if len(sys.argv) > 1 else 384
B = np.load(sys.argv[2]) if len(sys.argv) > 2 else np.tril(np.random.default_rng(d).standard_normal((d, d))) * (0.97 ** np.arange(d))
B = torch.from_numpy(np.ascontiguousarray(B)).cuda()
Ub = torch.empty((d, d), dtype=torch.float64, device="cuda"); Vb = torch.empty_like(Ub)
S = torch.empty(d, dtype=torch.float64, device="cuda")
print("sweeps", T.dbg_small_svd(B, Ub, S, Vb))
