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


PROBE_PHASE = {"nn": "ortho_nn", "tn": "ortho_tn", "spmm": "apply_A:csr",
               "dense_nn": "apply_A:dense", "dense_tn": "apply_AT:dense"}


def write_launch_summary(lpath, out_md, tag, what):
    agg = launch_summary(lpath)
    tot = sum(v[1] for v in agg.values())
    with open(out_md, "w") as f:
        f.write(f"# ncu launch list summary ({tag})\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over "
                f"`{what}` (handle creation + one solve + the untimed residual check). "
                "Per-launch times are cold-cache and serialised: compare shares.\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |\n")


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    for fn in sorted(os.listdir(src)):
        m = re.fullmatch(r"launches(_(\w+?)_(lanczos|rsvd))?\.csv", fn)
        if not m:
            continue
        suffix = f"_{m.group(2)}_{m.group(3)}" if m.group(1) else ""
        shutil.copy(os.path.join(src, fn), os.path.join(prof, f"{tag}{suffix}_launches.csv"))
        what = (f"bench.py --config {m.group(2)} --algo {m.group(3)} --steps 1 --warmup 0"
                if m.group(1) else "bench.py --steps 1 --warmup 0")
        write_launch_summary(os.path.join(src, fn),
                             os.path.join(prof, f"{tag}{suffix}_launch_summary.md"), tag, what)
    full = {}
    for fn in sorted(os.listdir(src)):
        if fn.startswith("full_") and fn.endswith(".ncu-rep"):
            m = full_metrics(os.path.join(src, fn))
            if m:
                full[fn[5:-8]] = m
    # traffic probes: one launch at a known shape (scripts/traffic_probe.py)
    tfile = os.path.join(prof, "ncu_traffic.json")
    traffic = json.load(open(tfile)) if os.path.exists(tfile) else {}
    for fn in sorted(os.listdir(src)):
        m = re.fullmatch(r"traffic_(\w+)\.ncu-rep", fn)
        if not m:
            continue
        mode = m.group(1)
        probe = None
        for ext in ("json", "err"):  # ncu may route the probe's stdout to either
            fp = os.path.join(src, f"traffic_{mode}.{ext}")
            if os.path.exists(fp):
                for ln in open(fp):
                    if ln.startswith('{"mode"'):
                        probe = json.loads(ln)
        if probe is None:
            continue
        met = full_metrics(os.path.join(src, fn))
        if not met or "dram__bytes_read.sum" not in met:
            continue
        dram = to_bytes(met["dram__bytes_read.sum"]) + to_bytes(met["dram__bytes_write.sum"])
        full[f"traffic_{mode}"] = met
        traffic[PROBE_PHASE[mode]] = {
            "kernel": met["kernel"][:80], "probe": probe, "dram_bytes": dram,
            "alg_bytes": probe["alg_bytes"], "dram_over_alg": round(dram / probe["alg_bytes"], 4),
            "source": f"profiles/{tag}_ncu_full.json (traffic_{mode})"}
    traffic["_doc"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one `ncu --set full` "
                       "launch at a known shape (scripts/traffic_probe.py) divided by that "
                       "launch's ALGORITHMIC bytes (DESIGN.md section 6); bench.py multiplies the "
                       "ratio by the phase's average algorithmic bytes per launch to report "
                       "roofline.traffic.")
    with open(tfile, "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(prof, f"{tag}_ncu_full.json"), "w") as f:
        json.dump(full, f, indent=1)
    print(json.dumps(full, indent=1))


if __name__ == "__main__":
    main()
