"""Round-2 ncu evidence -> profiles/r02/ (run here after the gpurun session of
scripts/gpu_session.sh brought back gpurun_out/r02_*):

  profiles/r02/C2_launches.csv, C2_launch_summary.md   the launch list of one C2
      solve (gpu__time_duration per launch; cold-cache, serialised: compare shares)
  profiles/r02/ncu_full_key_metrics.json   key metrics of each --set full capture
  profiles/ncu_traffic_bench.json          (via scripts/capture_traffic.py) DRAM bytes
      per launch of the benched ortho_nn / ortho_tn kernels, read by bench.py
"""
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from summarize_ncu import launch_summary  # noqa: E402

G = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles", "r02")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum"]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "selected", "not_selected", "branch_resolving",
          "dispatch_stall", "membar", "no_instruction"]


def full_metrics(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")][:100] if "Kernel Name" in hdr else "?"}
        for k in KEYS:
            if k in hdr:
                rec[k] = r[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        st = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in hdr and r[hdr.index(k)] not in ("", "0"):
                st[s] = int(float(r[hdr.index(k)].replace(",", "")))
        tot = sum(st.values()) or 1
        rec["stall_samples_share"] = {k: round(v / tot, 3) for k, v in
                                      sorted(st.items(), key=lambda kv: -kv[1])}
        out.append(rec)
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    lp = os.path.join(G, "r02_C2_launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(OUT, "C2_launches.csv"))
        agg = launch_summary(lp)
        tot = sum(v[1] for v in agg.values())
        lines = ["# C2 launch list (ncu gpu__time_duration, one solve incl. handle creation)",
                 "", f"total {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches", "",
                 "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {t / 1e3:.3f} | {t / tot:.3f} |")
        open(os.path.join(OUT, "C2_launch_summary.md"), "w").write("\n".join(lines) + "\n")
    full = {}
    for f in sorted(os.listdir(G)):
        m = re.match(r"r02_full_(.+)_raw\.csv$", f)
        if m:
            full[m.group(1)] = full_metrics(os.path.join(G, f))
    json.dump(full, open(os.path.join(OUT, "ncu_full_key_metrics.json"), "w"), indent=1)
    for phase, kern in (("ortho_nn", "gemm_nn_tma_kernel"), ("ortho_tn", "gemm_tn_tma_kernel")):
        p = os.path.join(G, f"r02_traffic_{phase}.csv")
        if os.path.exists(p):
            shutil.copy(p, os.path.join(OUT, f"traffic_{phase}.csv"))
            subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "capture_traffic.py"),
                            phase, kern, os.path.join(OUT, f"traffic_{phase}.csv")], check=True)
    for f in ("r02_full_nn_sass.csv",):
        if os.path.exists(os.path.join(G, f)):
            shutil.copy(os.path.join(G, f), os.path.join(OUT, f.replace("r02_", "")))


if __name__ == "__main__":
    main()
