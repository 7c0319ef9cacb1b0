"""Where the end-to-end (host buffers) time of a C2 solve goes.
    python scripts/e2e_breakdown.py"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import CONFIGS, SEEDS, powerlaw_csr  # noqa: E402

cfg = CONFIGS["C2"]
m, n = cfg["m"], cfg["n"]
csr = powerlaw_csr(m, n, cfg["nnz"], cfg["alpha"], SEEDS["C2"])
pinned = tuple(torch.from_numpy(x).pin_memory() for x in csr)
T.lib()
torch.cuda.synchronize()


def run(inp, label, out_pinned):
    t0 = time.perf_counter()
    h = T.TruncatedSVD(csr=inp, shape=(m, n))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    h.set_seed(SEEDS["C2"]); h.set_krylov_dim(cfg["d"])
    h.block_lanczos(cfg["r"], cfg["b"], cfg["tol"], cfg["maxit"])
    torch.cuda.synchronize(); t2 = time.perf_counter()
    if out_pinned:
        U = torch.empty((m, cfg["r"]), dtype=torch.float64).pin_memory()
        V = torch.empty((n, cfg["r"]), dtype=torch.float64).pin_memory()
        S = torch.empty(cfg["r"], dtype=torch.float64).pin_memory()
        t2 = time.perf_counter()
        h.get_into(U.numpy(), S.numpy(), V.numpy())
    else:
        h.get()
    t3 = time.perf_counter()
    h.close()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"{label}: create {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms  get {1e3*(t3-t2):.1f} ms  "
          f"destroy {1e3*(t4-t3):.1f} ms  total {1e3*(t4-t0):.1f} ms", flush=True)


for i in range(3):
    run(csr, f"pageable #{i}", False)
for i in range(3):
    run(tuple(x.numpy() for x in pinned), f"pinned   #{i}", True)
