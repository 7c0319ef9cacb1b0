#!/bin/bash
# Evidence for the next round: C3 (b = 32, DMMA-bound passes) ncu full captures + stall summary.
mkdir -p gpurun_out/c3
B="python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
for K in "gemm_nn_tma_kernel:40" "gemm_tn_tma_kernel:40" "jacobi_reg_kernel:0"; do
  N=${K%%:*}; S=${K##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$N -s $S -c 1 -o gpurun_out/c3/full_$N $B > /dev/null 2>&1
  echo "$N rc=$?"
done
python - <<'PY'
import csv, io, json, subprocess, glob
out = {}
for rep in sorted(glob.glob('gpurun_out/c3/*.ncu-rep')):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3: continue
    h, u, v = r[0], r[1], r[2]
    d = {}
    for k, uu, vv in zip(h, u, v):
        if k in ('Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
                 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
                 'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active',
                 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
                 'smsp__average_warp_latency_per_inst_issued.ratio') or (
                 'smsp__average_warps_issue_stalled' in k and k.endswith('_per_issue_active.ratio')):
            try:
                if k != 'Kernel Name' and float(vv) < 0.05: continue
            except ValueError:
                pass
            d[k] = (vv + ' ' + uu).strip()
    out[rep.split('/')[-1][:-8]] = d
json.dump(out, open('gpurun_out/c3/C3_ncu_full.json', 'w'), indent=1)
print(json.dumps(out, indent=1)[:3000])
PY
rm -f gpurun_out/c3/*.ncu-rep
