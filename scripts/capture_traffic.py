"""DRAM traffic of the benched launches (bench.py roofline.traffic).

Run on the GPU box (one GPU, never under torchrun):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:<kernel> --csv --log-file gpurun_out/traffic_<phase>.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0
    python scripts/capture_traffic.py <phase> <kernel> gpurun_out/traffic_<phase>.csv

writes profiles/ncu_traffic_bench.json[<phase>] = mean dram_bytes_read +
dram_bytes_write per launch of that kernel over the whole C2 solve (the
same command bench.py times), which bench.py reports as roofline.traffic
(bytes per launch, like roofline.achieved).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(phase, kernel, path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = {}
    for r in rows:
        if "Metric Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        rec = dict(zip(hdr, r))
        if kernel not in rec.get("Kernel Name", ""):
            continue
        key = rec["ID"]
        val = float(rec["Metric Value"].replace(",", ""))
        unit = rec.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                 "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1.0)
        per.setdefault(key, {})[rec["Metric Name"]] = val * scale
    launches = [v for v in per.values() if "dram__bytes_read.sum" in v]
    if not launches:
        raise SystemExit(f"no launches of {kernel} in {path}")
    n = len(launches)
    dram = sum(v["dram__bytes_read.sum"] + v.get("dram__bytes_write.sum", 0.0) for v in launches)
    t = sum(v.get("gpu__time_duration.sum", 0.0) for v in launches)
    out_p = os.path.join(ROOT, "profiles", "ncu_traffic_bench.json")
    data = json.load(open(out_p)) if os.path.exists(out_p) else {}
    data[phase] = {"kernel": kernel, "launches": n, "dram_bytes_per_launch": dram / n,
                   "ncu_time_s_per_launch": t / n,
                   "source": f"{os.path.relpath(path, ROOT)}: ncu --metrics dram__bytes_read.sum,"
                             "dram__bytes_write.sum on every launch of one C2 solve "
                             "(bench.py --steps 1 --warmup 0)"}
    json.dump(data, open(out_p, "w"), indent=1)
    print(json.dumps(data[phase]))


if __name__ == "__main__":
    main(*sys.argv[1:4])
