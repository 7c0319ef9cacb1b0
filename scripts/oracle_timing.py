"""Host-oracle timing on the GPU box: one complete oracle
LancSVD solve per config, with 1 BLAS thread and with all cores, plus the
host facts (nproc, CPU model, RAM).  The oracle is never tuned for this.

    python scripts/oracle_timing.py [C2 C4 ...] > profiles/<round>_oracle_timing.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from threadpoolctl import threadpool_limits  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
from tsvd_inputs import SEEDS  # noqa: E402


def main():
    cfgs = sys.argv[1:] or ["C2", "C4"]
    out = {"host": bench.host_info(), "runs": []}
    for name in cfgs:
        cfg, _, work = bench.make_workload(name, 0)
        op = oracle.Operator(dense=work["A"]) if "A" in work else \
            oracle.Operator(csr=work["csr"], shape=work["shape"])
        for threads in (os.cpu_count(), 1):
            with threadpool_limits(threads):
                t0 = time.perf_counter()
                res = oracle.lancsvd(op, cfg["r"], cfg["b"], cfg["d"], cfg["tol"], cfg["maxit"],
                                     SEEDS[name])
                t = time.perf_counter() - t0
            rec = {"config": name, "threads": threads, "seconds": round(t, 2),
                   "cycles": res.cycles, "nconv": res.nconv, "r": cfg["r"]}
            out["runs"].append(rec)
            print(json.dumps(rec), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
