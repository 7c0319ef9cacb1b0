#!/bin/bash
# Round evidence: official bench line, reference arm, ncu launch list and
# full-set captures of the top kernels.  Run under gpurun from the repo root.
#   bash scripts/profile_round.sh [CONFIG] [ALGO]
set -x
CFG=${1:-C2}
ALGO=${2:-lanczos}
OUT=gpurun_out
mkdir -p $OUT
B="python bench.py --config $CFG --algo $ALGO"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
$B > $OUT/bench_${CFG}_${ALGO}.json 2> $OUT/bench_${CFG}_${ALGO}.err
$B --impl reference --steps 1 --warmup 0 > $OUT/bench_ref_${CFG}_${ALGO}.json 2> $OUT/bench_ref_${CFG}_${ALGO}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $OUT/launches_${CFG}_${ALGO}.csv \
    $B --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for K in ${KERNELS:-"gemm_nn_tma_kernel:60" "gemm_tn_tma_kernel:60" "spmm_kernel:20" "rowT_kernel:40" "jacobi_reg_kernel:0"}; do
  N=${K%%:*}; S=${K##*:}
  ncu --set full --import-source on --clock-control none -k regex:$N -s $S -c 1 \
      -o $OUT/full_${CFG}_${ALGO}_$N \
      $B --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
ls -la $OUT
