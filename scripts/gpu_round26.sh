#!/bin/bash
# Round evidence on the final code: official C2 line (+ cpu baseline, e2e), reference arm,
# ncu launch list + full captures, DRAM-traffic probes at known shapes.
mkdir -p gpurun_out
bash scripts/profile_round.sh C2 lanczos > gpurun_out/profile_round.log 2>&1
for P in "nn:gemm_nn_tma_kernel" "tn:gemm_tn_tma_kernel" "spmm:spmm_kernel" "dense_nn:gemm_nn_tma_kernel" "dense_tn:gemm_tn_tma_kernel"; do
  M=${P%%:*}; K=${P##*:}
  timeout 600 ncu --set full --clock-control none -k regex:$K -c 1 -o gpurun_out/traffic_$M \
      python scripts/traffic_probe.py $M > gpurun_out/traffic_$M.json 2>&1
  echo "traffic $M rc=$?"
done
python -c "
import json
d=json.loads(open('gpurun_out/bench_C2_lanczos.json').read().strip().splitlines()[-1])
print('C2 TTS', d['value'], d['e2e'], d['roofline'], d['cpu_baseline'], d['clocks'], d['gpu_launches'])
"
tail -1 gpurun_out/bench_ref_C2_lanczos.json | cut -c1-300
ls gpurun_out
# keep what comes back under 64 MiB: summaries + two full reports
python scripts/summarize_ncu.py r01f gpurun_out > /dev/null
mkdir -p gpurun_out/evid
cp profiles/r01f_* profiles/ncu_traffic.json gpurun_out/evid/
mkdir -p gpurun_out/keep
mv gpurun_out/full_C2_lanczos_gemm_nn_tma_kernel.ncu-rep gpurun_out/full_C2_lanczos_spmm_kernel.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
