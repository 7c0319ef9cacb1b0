"""Times the device G1 generator stage by stage (development probe)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tsvd_inputs as ti

for (m, nnz) in [(1_000_000, 10_000_000), (50_000_000, 1_000_000_000)]:
    torch.cuda.synchronize()
    t = time.time()
    out = ti.powerlaw_csr_device(m, m, nnz, 2.5, seed=0x2403062185)
    torch.cuda.synchronize()
    L = torch.diff(out[0])
    print(f"m={m} nnz={out[1].numel()} {time.time() - t:.1f} s  max row {int(L.max())} "
          f"peak {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
    del out, L
    torch.cuda.empty_cache()
