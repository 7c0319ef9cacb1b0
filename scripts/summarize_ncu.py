"""Summarise a round's ncu evidence (gpurun_out/) into profiles/<tag>_*.

    python scripts/summarize_ncu.py r01 [gpurun_out]

Writes:
  profiles/<tag>_launches.csv      the raw ncu launch list (gpu__time_duration per launch)
  profiles/<tag>_launch_summary.md per-kernel totals and shares of the captured solve
  profiles/<tag>_ncu_full.json     key metrics of each `ncu --set full` capture
  profiles/ncu_traffic.json        dram bytes / algorithmic bytes of the dominant phase
                                   kernel (read by bench.py for roofline.traffic)
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "s": 1e6, "second": 1e6}
    for r in rows[hdr + 1:]:
        if len(r) <= iv:
            continue
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("tsvd::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    return agg


FULL_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
    "launch__grid_size", "sm__cycles_elapsed.avg.per_second",
]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return None
    h, units, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for k in FULL_KEYS:
        if k in h:
            i = h.index(k)
            d[k] = f"{v[i]} {units[i]}".strip()
    return d


def to_bytes(s):
    val, unit = s.split()[0], (s.split()[1] if len(s.split()) > 1 else "byte")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(val.replace(",", "")) * mult


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    lpath = os.path.join(src, "launches.csv")
    if os.path.exists(lpath):
        shutil.copy(lpath, os.path.join(prof, f"{tag}_launches.csv"))
        agg = launch_summary(lpath)
        tot = sum(v[1] for v in agg.values())
        with open(os.path.join(prof, f"{tag}_launch_summary.md"), "w") as f:
            f.write(f"# ncu launch list summary ({tag})\n\n")
            f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over "
                    "`bench.py --steps 1 --warmup 0` (handle creation + one C2 solve). "
                    "Per-launch times are cold-cache and serialised: compare shares.\n\n")
            f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |\n")
    full = {}
    for fn in sorted(os.listdir(src)):
        if fn.startswith("full_") and fn.endswith(".ncu-rep"):
            m = full_metrics(os.path.join(src, fn))
            if m:
                full[fn[5:-8]] = m
    with open(os.path.join(prof, f"{tag}_ncu_full.json"), "w") as f:
        json.dump(full, f, indent=1)
    print(json.dumps(full, indent=1))


if __name__ == "__main__":
    main()
