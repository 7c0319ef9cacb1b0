#!/usr/bin/env python
"""Benchmark: truncated-SVD time-to-solution on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A "step" is one complete tsvd_block_lanczos solve (all SURVEY 8(a) rows:
Philox start block + CholQR2, per block step A^T.Qbar (CSR(A^T) SpMM),
CGS-CQR2 against P, A.Q (CSR SpMM), CGS-CQR2 against Pbar, B_k assembly,
one-sided Jacobi SVD of B_k, rho test, restart, outputs U, V, sign) on the
synthetic config's CSR matrix, with A already resident in HBM.  value = the
time-to-solution in seconds (lower is better), max over ranks.

N > 1 (torchrun, one process per GPU): the SAME workload is solved once,
row-partitioned across the ranks (nnz-balanced row split,
NCCL reduce-scatter of A^T Qbar, all-gather of Q_i, all-reduced projections
and Grams); "scaling": "strong", value = max over ranks of the solve time.
The default workload at N > 1 is C5 (m = n = 5e7, nnz 1e9, fixed work: one
cycle at d = 160), the config north_star's 1 -> 8 GPU scaling is defined on;
`--config C5` gives its N = 1 point.

--impl reference: the CPU oracle (oracle/, numpy/scipy fp64) on the host
cores, rank 0 only.  C1, C2, C4: every step is one complete oracle solve,
timed end to end (no extrapolation); steps stop after --ref-budget seconds
(>= 1 step) and the line reports the steps actually run.  C3 / C5 (minutes /
150 GB on the host): a bounded sample of block steps extrapolated linearly
in the block index (labelled as such in `sample`).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "truncated-SVD time-to-solution (s) at fixed residual; SpMM/QR HBM GB/s vs peak"
CONFIG_TEXT = {
    "C1": "dense 200x100 FP64 with prescribed geometric spectrum, r=10, block Lanczos b=4",
    "C2": "synthetic sparse square CSR, m=n=1e6, nnz~1e7, power-law row lengths, r=50, "
          "block Lanczos b=16 on 1 B200",
    "C3": "synthetic sparse rectangular CSR, m=4e6, n=5e5, nnz~5e7, r=100, block Lanczos b=32",
    "C4": "synthetic dense 40000x20000 FP64 with slowly decaying spectrum, r=200, "
          "block Lanczos b=32",
    "C5": "large synthetic sparse CSR, m=n=5e7, nnz~1e9, r=100, b=32; fixed work: one "
          "restart cycle at d=160 (SURVEY 8(d) C5 (i))",
    "C5g2": "G2 twin of C5: block-diagonal CSR m=n=5e7, nnz~1e9, closed-form spectrum (top 100 "
            "in [100, 200], tail <= 20), r=100, b=32, d=160, thick restart keep 128, tol 1e-8 "
            "(SURVEY 8(d) C5 (iii))",
}


def _fp64_peak():
    """FP64 DMMA (mma.sync m8n8k4 f64) peak measured on this pool's B200 by
    scripts/peaks.cu (profiles/box_facts_r01.json); MEASURED_PEAKS.json has no
    FP64 entry and tcgen05 has no f64 kind."""
    try:
        with open(os.path.join(ROOT, "profiles", "box_facts_r01.json")) as f:
            return float(json.load(f)["dmma_m8n8k4_f64_tflops"]), \
                "profiles/box_facts_r01.json dmma_m8n8k4_f64_tflops (measured, scripts/peaks.cu)"
    except Exception:
        return 37.0, "fallback 37 TF/s (FP64 DMMA)"


def workload_text(cfg_name: str, algo: str) -> str:
    from tsvd_inputs import CONFIGS
    t = CONFIG_TEXT.get(cfg_name, "")
    if algo == "rsvd":
        c = CONFIGS[cfg_name]
        t = t.split(", block Lanczos")[0] + f", rSVD p={c['rsvd_p']} q={c['rsvd_q']}"
    return f"{cfg_name}: {t}"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------- workload --
def make_workload(cfg_name: str, rank: int = 0):
    from tsvd_inputs import CONFIGS, SEEDS, dense_prescribed, powerlaw_csr, spectrum_eq16
    cfg = dict(CONFIGS[cfg_name])
    seed = SEEDS[cfg_name] + 1000 * rank
    if cfg.get("device_gen") == "g2":  # C5 (iii): G2 twin, closed-form spectrum, in HBM
        import numpy as np
        from tsvd_inputs import blockdiag_csr_device
        t0 = time.time()
        hi, lo, k = cfg["top"]
        rp, ci, va, sig = blockdiag_csr_device(cfg["m"], cfg["n"], cfg["mean_block"],
                                               cfg["alpha"], seed, np.linspace(hi, lo, k),
                                               tail_max=cfg["tail_max"])
        print(f"{cfg_name}: generated {ci.numel()} nonzeros (G2) in HBM in "
              f"{time.time() - t0:.1f} s", file=sys.stderr, flush=True)
        return cfg, seed, dict(csr=(rp, ci, va), shape=(cfg["m"], cfg["n"]), sigma=sig[:k + 1])
    if cfg.get("device_gen"):  # C5: 1e9 nonzeros, generated in HBM (tsvd_inputs)
        from tsvd_inputs import powerlaw_csr_device
        t0 = time.time()
        csr = powerlaw_csr_device(cfg["m"], cfg["n"], cfg["nnz"], cfg["alpha"], seed)
        print(f"{cfg_name}: generated {csr[1].numel()} nonzeros in HBM in {time.time() - t0:.1f} s",
              file=sys.stderr, flush=True)
        return cfg, seed, dict(csr=csr, shape=(cfg["m"], cfg["n"]))
    if cfg["kind"] == "csr":
        csr = powerlaw_csr(cfg["m"], cfg["n"], cfg["nnz"], cfg["alpha"], seed)
        return cfg, seed, dict(csr=csr, shape=(cfg["m"], cfg["n"]))
    s = spectrum_eq16(cfg["n"])
    refl = None if cfg["m"] * cfg["n"] <= 4_000_000 else 4
    A = dense_prescribed(cfg["m"], cfg["n"], s, seed, n_reflectors=refl)
    return cfg, seed, dict(A=A)


def shard_workload(work, rank, world, T):
    """This rank's rows (nnz-balanced split by the library's partitioner)."""
    import numpy as np
    if "csr" in work:
        rp, ci, va = work["csr"]
        m, n = work["shape"]
        rp_h = rp.cpu().numpy() if hasattr(rp, "cpu") else rp
        b = T.partition_rows(rp_h, world)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        lo, hi = int(rp_h[r0]), int(rp_h[r1])
        if hasattr(rp, "cpu"):  # device-generated (C5): every rank built the same bytes
            local = dict(csr=((rp[r0:r1 + 1] - lo).contiguous(), ci[lo:hi].clone(),
                              va[lo:hi].clone()))
        else:
            local = dict(csr=(np.ascontiguousarray(rp[r0:r1 + 1] - lo), ci[lo:hi], va[lo:hi]))
    else:
        A = work["A"]
        m, n = A.shape
        b = np.linspace(0, m, world + 1).astype(np.int64)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        local = dict(A=np.ascontiguousarray(A[r0:r1]))
    return local, dict(m_global=m, n_global=n, row_begin=r0, row_end=r1)


def _to_device(work):
    import numpy as np
    import torch
    out = dict(work)
    if "csr" in work:
        out["csr"] = tuple(x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x)).cuda()
                           for x in work["csr"])
    else:
        out["A"] = torch.from_numpy(work["A"]).cuda()
    return out


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------- cpu baseline --
_HOST_WORK = {}


def host_workload(cfg_name: str):
    """make_workload for the host oracle, generated once per process (the
    reference arm runs several steps on the same bytes)."""
    if cfg_name not in _HOST_WORK:
        _HOST_WORK.clear()
        _HOST_WORK[cfg_name] = make_workload(cfg_name, 0)
    return _HOST_WORK[cfg_name]


def oracle_sample(cfg_name: str, budget_s: float, cycles: int, seed: int, keep: int = 0,
                  d: int | None = None):
    """Time the oracle's LancSVD block steps (Alg. 2 S2-S5, calling only
    oracle/) for ~budget_s on the host, fit t_i = a + c*i and extrapolate to
    `cycles` full cycles of k = d/b steps plus the small SVD."""
    import numpy as np
    from threadpoolctl import threadpool_info
    import oracle
    from oracle.core import DrawCtx, cholqr2, cgs_cqr2, small_svd
    scale = 1.0
    if cfg_name == "C5":  # host-sized sample: C5 scaled down 10x (same alpha, mean row)
        cfg_name, scale = "C5s", 10.0
    cfg, seed_, work = host_workload(cfg_name)
    op = oracle.Operator(dense=work["A"]) if "A" in work else oracle.Operator(csr=work["csr"], shape=work["shape"])
    m, n, b = cfg["m"], cfg["n"], cfg["b"]
    d = d or cfg["d"]
    k = d // b
    ctx = DrawCtx(seed)
    t0 = time.perf_counter()
    Qbar, _ = cholqr2(oracle.gaussian_block(m, b, seed, draw=0), ctx)
    t_start = time.perf_counter() - t0
    Pbar = np.zeros((m, d + b))
    P = np.zeros((n, d))
    Pbar[:, :b] = Qbar
    times = []
    t_begin = time.perf_counter()
    for i in range(k):
        ts = time.perf_counter()
        lo, hi = i * b, (i + 1) * b
        Y = op.rmatmul(Pbar[:, lo:hi])
        Q = cholqr2(Y, ctx)[0] if i == 0 else cgs_cqr2(Y, P[:, :lo], ctx)[0]
        P[:, lo:hi] = Q
        Z = op.matmul(Q)
        Pbar[:, hi:hi + b] = cgs_cqr2(Z, Pbar[:, :hi], ctx)[0]
        times.append(time.perf_counter() - ts)
        if time.perf_counter() - t_begin > budget_s and len(times) >= 3:
            break
    ts = time.perf_counter()
    small_svd(np.random.default_rng(0).standard_normal((d, d)))
    t_svd = time.perf_counter() - ts
    idx = np.arange(len(times))
    c, a = np.polyfit(idx, np.array(times), 1) if len(times) > 1 else (0.0, times[0])
    def t_of(i):
        return max(a + c * i, times[0] * 0.5)
    per_cycle = float(sum(t_of(i) for i in range(k))) + t_svd
    if keep:  # thick restart: later cycles run steps keep/b .. k-1 (+ restart products)
        later = float(sum(t_of(i) for i in range(keep // b, k))) + t_svd + t_of(k - 1)
        est = t_start + per_cycle + (cycles - 1) * later
    else:
        est = t_start + cycles * per_cycle
    est *= scale  # every step is linear in m, n and nnz at fixed d, b
    threads = max((x.get("num_threads", 1) for x in threadpool_info()), default=1)
    sample = (f"{cfg_name} LancSVD block steps i=0..{len(times)-1} of k={k} of cycle 1 "
              f"({sum(times):.1f} s measured) + SVD({d}) ({t_svd:.2f} s); t_i fitted "
              f"linearly in i and extrapolated to {cycles} cycle(s) x {k} steps"
              + (f" (thick restart: cycles > 1 run steps {keep // b}..{k - 1})" if keep else "")
              + (f"; x{scale:g} for C5 (linear in m, n, nnz at fixed d, b)" if scale != 1.0 else ""))
    return dict(value=est, unit="s", cores=int(threads), kind="oracle", sample=sample,
                measured_s=sum(times) + t_svd + t_start)


def host_info():
    """The host the oracle runs on (nproc / lscpu / RAM)."""
    info = {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["cpu"] = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            info["mem_gb"] = round(int(f.readline().split()[1]) / 1e6, 1)
    except OSError:
        pass
    return info


def oracle_threads():
    from threadpoolctl import threadpool_info
    return int(max((x.get("num_threads", 1) for x in threadpool_info()), default=1))


# full oracle solves that finish in well under a minute on the box's host
FULL_ORACLE = {"C1", "C2", "C4"}


def oracle_full(cfg_name: str, seed: int, keep: int = 0, d: int | None = None,
                maxit: int | None = None):
    """One complete oracle LancSVD solve (Alg. 2, oracle/lancsvd.py) of the
    config on the host, timed end to end (matrix already in host memory, as
    the GPU arm's A is resident in HBM).  No extrapolation."""
    import oracle
    cfg, _, work = host_workload(cfg_name)
    op = oracle.Operator(dense=work["A"]) if "A" in work else \
        oracle.Operator(csr=work["csr"], shape=work["shape"])
    d = d or cfg["d"]
    maxit = maxit or cfg["maxit"]
    t0 = time.perf_counter()
    res = oracle.lancsvd(op, cfg["r"], cfg["b"], d, cfg["tol"], maxit, seed, keep=keep)
    t = time.perf_counter() - t0
    sample = (f"{cfg_name} complete oracle LancSVD solve (r={cfg['r']}, b={cfg['b']}, d={d}, "
              f"tol={cfg['tol']}, maxit={maxit}{f', keep={keep}' if keep else ''}): "
              f"{res.cycles} cycle(s), {res.nconv}/{cfg['r']} converged, measured end to end "
              f"(no extrapolation)")
    return dict(value=t, unit="s", cores=oracle_threads(), kind="oracle", sample=sample,
                host=host_info(), measured_s=t, cycles=res.cycles, nconv=res.nconv)


def oracle_sample_rsvd(cfg_name: str, budget_s: float, seed: int):
    """Time the oracle's RandSVD (Alg. 1, calling only oracle/) on the host:
    power iterations S1-S4 are run until ~budget_s has passed (at least one),
    their mean time is extrapolated to the q+1 iterations of the config, plus
    the small SVD of R_p and the output products S6-S7 (run once)."""
    import numpy as np
    from threadpoolctl import threadpool_info
    import oracle
    from oracle.core import DrawCtx, cgs_qr, small_svd
    from oracle.philox import gaussian_block
    cfg, _, work = host_workload(cfg_name)
    op = oracle.Operator(dense=work["A"]) if "A" in work else oracle.Operator(csr=work["csr"], shape=work["shape"])
    n, r, p, q = cfg["n"], cfg["r"], cfg["rsvd_p"], cfg["rsvd_q"]
    l, bq = r + p, 16
    ctx = DrawCtx(seed)
    Q = gaussian_block(n, l, seed, draw=0)
    its = []
    t_begin = time.perf_counter()
    while True:
        ts = time.perf_counter()
        Qb, _ = cgs_qr(op.matmul(Q), bq, ctx)
        Q, R = cgs_qr(op.rmatmul(Qb), bq, ctx)
        its.append(time.perf_counter() - ts)
        if time.perf_counter() - t_begin > budget_s or len(its) >= q + 1:
            break
    ts = time.perf_counter()
    Ub, S, Vb = small_svd(R)
    _ = Qb @ Vb[:, :r], Q @ Ub[:, :r]
    t_tail = time.perf_counter() - ts
    est = (q + 1) * float(np.mean(its)) + t_tail
    threads = max((x.get("num_threads", 1) for x in threadpool_info()), default=1)
    sample = (f"{cfg_name} RandSVD l={l}, b_qr={bq}: {len(its)} of {q + 1} power iterations "
              f"measured ({sum(its):.1f} s) + SVD(R_p) and outputs ({t_tail:.2f} s); mean "
              f"iteration time extrapolated to q+1 = {q + 1}")
    return dict(value=est, unit="s", cores=int(threads), kind="oracle", sample=sample,
                measured_s=sum(its) + t_tail)


def residual_check(h, U=None, V=None):
    """Acceptance numbers of the returned triplets (not timed): e_i =
    ||A v_i - sigma_i u_i|| / sigma_1 (Eq. 14 as corrected, reading R13) by
    the library itself (tsvd_residuals: its own A.X and column norms,
    SURVEY 8(a) a17); the orthogonality of U, V (when they were copied out)
    by a torch matmul."""
    import numpy as np
    import torch
    e, R = h.residuals()
    out = {"e_max": float(e.max()), "e_median": float(np.median(e)), "R_max": float(R.max()),
           "by": "tsvd_residuals (library kernels)"}
    if U is not None:
        I = torch.eye(U.shape[1], dtype=U.dtype, device=U.device)
        out["UtU_minus_I_max"] = float((U.T @ U - I).abs().max())
        out["VtV_minus_I_max"] = float((V.T @ V - I).abs().max())
    return out


# ------------------------------------------------------------------- main --
def same_workload_n1(cfg_name, world):
    """At N > 1 the default workload is C5 while the N = 1 default (the BENCH
    line) is C2; the one-GPU time of the SAME workload, from the committed
    profile written by `bench.py --config C5` (builder-measured, not this
    run), so a scaling series can be read against it."""
    if world <= 1:
        return None
    f = os.path.join(ROOT, "profiles", "r02s", f"bench_{cfg_name}_fixed_work.json")
    if not os.path.exists(f):
        return None
    try:
        d = json.load(open(f))
        return {"value": d["value"], "unit": d["unit"], "source": os.path.relpath(f, ROOT),
                "note": "one B200, measured by the builder with bench.py --config " + cfg_name}
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None,
                    help="C1..C5; default C2 at N = 1 (BASELINE configs[1]) and C5 (the "
                         "largest sparse config, fixed work d = 160) at N > 1")
    ap.add_argument("--algo", default="lanczos", choices=["lanczos", "rsvd"],
                    help="lanczos = tsvd_block_lanczos (default); rsvd = tsvd_rsvd(r, p, q) "
                         "with the config's oversampling p and power iterations q")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--keep", type=int, default=None,
                    help="thick restart keeping L Ritz pairs (SURVEY 8(f) N1); 0 = the paper's "
                         "restart (Alg. 2 S7); default: the config's setting")
    ap.add_argument("--d", type=int, default=None, help="override the config's Krylov dimension")
    ap.add_argument("--maxit", type=int, default=None, help="override the config's maxit")
    ap.add_argument("--ortho", default="cgs_cqr2", choices=["cgs_cqr2", "bcgs_pip2"],
                    help="block orthogonalisation: the paper's CGS-CQR2 (Alg. 5, default) or "
                         "BCGS-PIP+ (SURVEY 8(f) N2 ablation)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--prof-mode", default="dominant", choices=["dominant", "all", "none"],
                    help="phases whose events are recorded inside the timed region")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=120.0,
                    help="--impl reference: stop after the step that crosses this many seconds")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    multi = world > 1 or args.gpus > 1
    cfg_name = args.config or ("C5" if multi else "C2")

    if args.impl == "reference":
        if rank != 0:
            return 0
        from tsvd_inputs import CONFIGS, SEEDS
        cfg = CONFIGS[cfg_name]
        # Each step is one COMPLETE oracle solve where that finishes in well
        # under a minute (C1, C2, C4: measured, not extrapolated); the host
        # oracle is never tuned, so there is nothing to warm up beyond one run.
        # Steps stop once `--ref-budget` seconds are spent (at least one),
        # so the run ends within a few minutes whatever K is; the line
        # reports the steps actually run.  Other configs (C3: ~5 min, C5:
        # 150 GB) fall back to the bounded, extrapolated sample.
        vals, last = [], None
        t_begin = time.perf_counter()
        full = args.algo == "lanczos" and cfg_name in FULL_ORACLE
        budget = max(5.0, args.ref_budget / max(1, args.steps))
        for it in range(args.steps):
            if full:
                last = oracle_full(cfg_name, SEEDS[cfg_name])
            elif args.algo == "rsvd":
                last = oracle_sample_rsvd(cfg_name, budget, seed=SEEDS[cfg_name])
            else:
                last = oracle_sample(cfg_name, budget, cycles=1, seed=SEEDS[cfg_name])
            vals.append(last["value"])
            if time.perf_counter() - t_begin >= args.ref_budget:
                break
        v = statistics.median(vals)
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s",
               "n_gpus": args.gpus, "steps": len(vals), "warmup": 0,
               "steps_requested": args.steps, "warmup_requested": args.warmup,
               "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": workload_text(cfg_name, args.algo), "algo": args.algo,
                          "m": cfg["m"], "n": cfg["n"], "r": cfg["r"], "b": cfg["b"],
                          "d": cfg["d"], "tol": cfg["tol"]},
               "cpu_baseline": {"value": v, "unit": "s", "cores": last["cores"],
                                "kind": "oracle", "sample": last["sample"],
                                "host": host_info(), "all_steps_s": [round(x, 3) for x in vals]},
               "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return 0

    import numpy as np
    import torch
    import paper_2403_06218_b200 as T

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    T.lib()

    cfg, seed, work = make_workload(cfg_name, 0)
    sigma_exact = work.pop("sigma", None)   # G2: the closed-form spectrum
    dist_kw = None
    # TSVD_BENCH_DIST=1 runs the row-partitioned NCCL path also with one rank
    use_dist = world > 1 or os.environ.get("TSVD_BENCH_DIST") == "1"

    def fresh_dist_kw(geo):
        # every NCCL communicator needs its own unique id (rank 0 -> broadcast)
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(T.nccl_unique_id()), dtype=torch.uint8))
        if dist:
            dist.broadcast(idt, 0)
        return dict(rank=rank, world=world, nccl_id=bytes(idt.cpu().numpy()), **geo)

    lwork = None
    if use_dist:
        lwork, geo = shard_workload(work, rank, world, T)
        dist_kw = fresh_dist_kw(geo)
        hwork = lwork
    else:
        hwork = dict(work)
    dwork = _to_device(hwork)
    if args.d is not None:
        cfg["d"] = args.d
    if args.keep is not None:
        cfg["keep"] = args.keep
    if args.maxit is not None:
        cfg["maxit"] = args.maxit
    keep = cfg.get("keep", 0)
    r, b, d, tol, maxit = cfg["r"], cfg["b"], cfg["d"], cfg["tol"], cfg["maxit"]
    stream = torch.cuda.current_stream()
    t0 = time.time()
    h = T.TruncatedSVD(**dwork, dist=dist_kw) if dist_kw else T.TruncatedSVD(**dwork)
    big = bool(cfg.get("device_gen"))
    if big:
        print(f"{cfg_name}: tsvd_create_csr {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
    nnz_total = int(work["csr"][1].numel() if big else len(work["csr"][1])) if "csr" in work else None
    if big:
        # C5: the library holds its own copies of A and CSR(A^T); free the
        # generator's so the d = 160 bases (141 GB) fit, and let the outputs be
        # formed in place (tsvd_set_output_mode AUTO)
        dwork = work = hwork = lwork = None
        torch.cuda.empty_cache()
        T.trim_memory(0)
        free, total = torch.cuda.mem_get_info()
        print(f"C5: A resident in the library, {free / 1e9:.1f} of {total / 1e9:.1f} GB free",
              file=sys.stderr, flush=True)
    h.set_seed(seed)
    h.set_krylov_dim(d)
    h.set_thick_restart(keep)
    h.set_ortho(args.ortho)
    rsvd = args.algo == "rsvd"
    if rsvd and "rsvd_p" not in cfg:
        raise SystemExit(f"config {cfg_name} has no rSVD settings")

    def solve(hh):
        if rsvd:
            return hh.rsvd(r, cfg["rsvd_p"], cfg["rsvd_q"])
        return hh.block_lanczos(r, b, tol, maxit)

    # the last warm-up solve records every phase (the per-phase breakdown,
    # untimed); the timed solves record only the dominant phase's events
    # (the roofline needs that phase's event time; every recorded phase call
    # adds two event records to the stream) -- --prof-mode all / none for A/B
    full_prof = None
    for it in range(args.warmup):
        t0 = time.time()
        last = it == args.warmup - 1
        if last:
            h.set_profiling(True)
            h.reset_profile()
        solve(h)
        if last:
            full_prof = h.profile()
            h.set_profiling(False)
        if big:
            torch.cuda.synchronize()
            print(f"{cfg_name}: warm-up solve {it}: {time.time() - t0:.1f} s {h.info()}",
                  file=sys.stderr, flush=True)
    dom_name = max(full_prof.items(), key=lambda kv: kv[1]["ms"])[0] if full_prof else None
    prof_names = list(T.PROF_PHASES)
    if args.prof_mode == "all" or dom_name is None:
        h.set_profiling(True)
    elif args.prof_mode == "dominant":
        h.set_profiling_mask(1 << prof_names.index(dom_name))
    else:
        h.set_profiling(False)
    h.reset_profile()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    gpu_idx = int(vis.split(",")[local]) if vis and vis.split(",")[local].isdigit() else local
    clocks = ClockSampler(gpu_idx)
    launches = 0
    infos = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        solve(h)
        inf = h.info()
        infos.append(inf)
        launches += int(inf["launches"])
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    prof = h.profile()
    h.set_profiling(False)
    if args.prof_mode != "all" and full_prof:
        timed_prof = prof
        prof = full_prof  # the breakdown; the roofline below uses the timed events
    else:
        timed_prof = prof
    accuracy = None
    if big:  # U, V (80 GB) stay in place in the bases; the library computes e
        accuracy = residual_check(h)
        if sigma_exact is not None:  # G2: sigma against the closed form
            import numpy as np
            S = h.singular_values()
            accuracy["sigma_err_max_over_sigma1"] = float(
                np.abs(S - sigma_exact[:len(S)]).max() / sigma_exact[0])
    else:
        U, S, V = h.get(device=True)
        accuracy = residual_check(h, U, V) if not use_dist else residual_check(h)
        del U, S, V
    h.close()

    # roofline of the dominant phase: the binding roof of its algorithmic work
    # -- HBM bytes vs the measured copy bandwidth, or FP64
    # flops vs the measured DMMA peak, whichever needs more time at peak
    peak, peak_kind = _peaks()
    fpeak, fpeak_src = _fp64_peak()
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    dn, dv = dom
    if timed_prof.get(dn, {}).get("calls", 0) > 0:
        dv = timed_prof[dn]  # event times of the dominant phase inside the timed region
    calls = max(1, dv["calls"])
    t_hbm = dv["bytes"] / (peak * 1e9) if dv["bytes"] > 0 else 0.0
    t_fp = dv["flops"] / (fpeak * 1e12) if dv["flops"] > 0 else 0.0
    traffic = None
    traffic_src = None
    # preferred: DRAM bytes per launch measured by ncu on the launches of this
    # very command (scripts/capture_traffic.py -> profiles/ncu_traffic_bench.json);
    # else the probe ratio at a known shape x this run's algorithmic bytes
    bfile = os.path.join(ROOT, "profiles", "ncu_traffic_bench.json")
    if cfg_name == "C2" and not rsvd and os.path.exists(bfile):
        try:
            tb = json.load(open(bfile)).get(dn)
            if tb:
                traffic, traffic_src = tb["dram_bytes_per_launch"], tb["source"]
        except Exception:
            traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if traffic is None and os.path.exists(tfile) and dv["bytes"] > 0:
        try:
            tj = json.load(open(tfile))
            tr = tj.get(f"{dn}:{'csr' if 'csr' in work else 'dense'}") or tj.get(dn)
            if tr:
                traffic = tr["dram_over_alg"] * dv["bytes"] / calls
                traffic_src = f"probe ratio {tr['dram_over_alg']} x alg bytes ({tr.get('source')})"
        except Exception:
            traffic = None
    sec = dv["ms"] * 1e-3
    if t_hbm == 0.0 and t_fp == 0.0:
        roof = {"bound": "alu", "kernel": dn, "achieved": None, "peak": None,
                "unit": "GFLOP/s", "frac": None, "traffic": None}
    elif t_fp > t_hbm:
        ach = dv["flops"] / sec / 1e12
        roof = {"bound": "tensor", "kernel": dn, "achieved": round(ach, 2), "peak": fpeak,
                "unit": "TFLOP/s", "frac": round(ach / fpeak, 4), "traffic": traffic,
                "alg_flops_per_launch": dv["flops"] / calls,
                "hbm_GBps": round(dv["bytes"] / sec / 1e9, 1),
                "peak_source": fpeak_src}
    else:
        ach = dv["bytes"] / sec / 1e9
        roof = {"bound": "hbm", "kernel": dn, "achieved": round(ach, 1), "peak": peak,
                "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": traffic,
                "fp64_TFps": round(dv["flops"] / sec / 1e12, 2),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
    roof["traffic_source"] = traffic_src
    roof["alg_bytes_per_launch"] = dv["bytes"] / calls
    roof["avg_launch_ms"] = dv["ms"] / calls
    total_ms = sum(v["ms"] for v in prof.values()) or 1.0
    prof_steps = 1 if prof is full_prof else args.steps
    phases = {k: {"ms_per_step": round(v["ms"] / prof_steps, 3),
                  "share": round(v["ms"] / total_ms, 4),
                  "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] > 0 and v["bytes"] > 0 else None,
                  "TFps": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] > 0 and v["flops"] > 0 else None,
                  "calls_per_step": v["calls"] / prof_steps}
              for k, v in prof.items() if v["calls"] > 0}

    # end-to-end through the public API with host buffers
    e2e = None
    if big:
        e2e = {"value": None, "unit": "s", "skipped": "C5: U, V alone are 80 GB of host copies"}
    elif args.e2e_steps > 0:
        torch.cuda.synchronize()
        times = []
        h2d = d2h = 0
        # inputs and results live in pinned host memory (allocated once, outside
        # the timed region); each step copies them in and out through the C ABI
        keep_alive = []

        def pinned(a):
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            keep_alive.append(t)
            return t.numpy()
        if "csr" in hwork:
            hin = dict(csr=tuple(pinned(x) for x in hwork["csr"]))
            h2d = sum(x.nbytes for x in hin["csr"])
        else:
            hin = dict(A=pinned(hwork["A"]))
            h2d = hin["A"].nbytes
        m_loc = int((geo["row_end"] - geo["row_begin"]) if use_dist else cfg["m"])
        n_loc = int(-(-cfg["n"] // world) if use_dist else cfg["n"])
        Uo, So, Vo = pinned(np.empty((m_loc, r))), pinned(np.empty(r)), pinned(np.empty((n_loc, r)))
        parts = []
        # one untimed step first (the device's memory pool regrows after the
        # timed handle was closed; early e2e steps showed 60-90 ms host-side
        # outliers), then the median of the timed ones
        for it in range(args.e2e_steps + 1):
            t0 = time.perf_counter()
            dkw2 = fresh_dist_kw(geo) if use_dist else None
            if "csr" in hin:
                h2 = (T.TruncatedSVD(csr=hin["csr"], dist=dkw2) if dkw2 else
                      T.TruncatedSVD(csr=hin["csr"], shape=hwork["shape"]))
            else:
                h2 = (T.TruncatedSVD(hin["A"], dist=dkw2) if dkw2 else T.TruncatedSVD(hin["A"]))
            t1 = time.perf_counter()
            h2.set_seed(seed)
            h2.set_krylov_dim(d)
            h2.set_thick_restart(keep)
            h2.set_ortho(args.ortho)
            solve(h2)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            h2.get_into(Uo[:h2.m], So, Vo[:h2.n])
            t3 = time.perf_counter()
            h2.close()
            torch.cuda.synchronize()
            if it == 0:
                continue
            times.append(time.perf_counter() - t0)
            parts.append([round(1e3 * (t1 - t0), 1), round(1e3 * (t2 - t1), 1),
                          round(1e3 * (t3 - t2), 1), round(1e3 * (time.perf_counter() - t3), 1)])
            d2h = Uo[:h2.m].nbytes + So.nbytes + Vo[:h2.n].nbytes
        ev = statistics.median(times)
        if dist:
            t = torch.tensor([ev], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ev = float(t.item())
        e2e = {"value": round(ev, 6), "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "steps_ms_create_solve_get_destroy": parts}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            if not rsvd and cfg_name in FULL_ORACLE:
                cpu = oracle_full(cfg_name, seed, keep=keep, d=d, maxit=maxit)
                cpu.pop("cycles", None)
                cpu.pop("nconv", None)
            else:
                cpu = (oracle_sample_rsvd(cfg_name, args.cpu_budget, seed=seed) if rsvd else
                       oracle_sample(cfg_name, args.cpu_budget, cycles=infos[-1]["cycles"],
                                     seed=seed, keep=keep, d=d))
                cpu["host"] = host_info()
            cpu.pop("measured_s", None)
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "error": repr(ex)}

    last = infos[-1]
    out = {
        "metric": METRIC, "value": round(ms / 1e3, 6), "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_text(cfg_name, args.algo), "algo": args.algo,
                   "m": cfg["m"], "n": cfg["n"], "nnz": nnz_total,
                   "r": r, "b": b, "d": d, "tol": tol, "maxit": maxit,
                   "restart": (f"thick, keep {keep} (SURVEY 8(f) N1)" if keep else
                               "paper (Alg. 2 S7)"),
                   "ortho": ("CGS-CQR2 (Alg. 5)" if args.ortho == "cgs_cqr2" else
                             "BCGS-PIP+ (SURVEY 8(f) N2 ablation)"),
                   "l2": "no flush: working set (A, A^T, bases) >> 126 MB L2",
                   "parallelism": f"row-partitioned x{world} (NCCL)" if world > 1 else "single"},
        "solver": {"cycles": last["cycles"], "nconv": last["nconv"], "rho_max": last["rho_max"],
                   "breakdowns": last["breakdowns"], "replaced": last["replaced"],
                   "sigma1": last["sigma1"]},
        "accuracy": accuracy,
        "roofline": roof,
        "phases": phases,
        "phases_from": ("the last warm-up solve, every phase recorded (untimed); the timed "
                        "solves record only the dominant phase" if prof is full_prof else
                        "the timed solves, every phase recorded"),
        "cpu_baseline": cpu,
        "same_workload_n1": same_workload_n1(cfg_name, world),
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
