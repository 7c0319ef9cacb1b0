#!/bin/bash
# Round evidence: official bench line, reference arm, ncu launch list and
# full-set captures of the top kernels.  Run under gpurun from the repo root.
set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for K in "gemm_nn_kernel:150" "gemm_tn_kernel:80" "spmm_short_kernel:40" "jacobi_reg_kernel:0"; do
  N=${K%%:*}; S=${K##*:}
  ncu --set full --import-source on --clock-control none -k regex:$N -s $S -c 1 -o $OUT/full_$N \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
ls -la $OUT
