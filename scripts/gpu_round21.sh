#!/bin/bash
# C5 evidence: bench line with the host-oracle sample, ncu launch list, full captures.
mkdir -p gpurun_out
nproc; free -g | head -2
timeout -s ABRT 1200 python -X faulthandler bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_C5.err | cut -c1-300
B="python bench.py --config C5 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_C5.csv $B > /dev/null 2>&1
echo "launch list rc=$?"
for K in "spmm_kernel:2" "gemm_nn_tma_kernel:8" "gemm_tn_tma_kernel:8" "rowT_kernel:10"; do
  N=${K%%:*}; S=${K##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$N -s $S -c 1 \
      -o gpurun_out/full_C5_$N $B > /dev/null 2>&1
  echo "$N rc=$?"
done
ls -la gpurun_out
