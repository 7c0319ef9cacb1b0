#!/bin/bash
# C3/C4 measurement + traffic probes (round 1, session 2)
set -x
OUT=gpurun_out; mkdir -p $OUT
for M in nn tn spmm dense_nn dense_tn; do
  case $M in nn) K=gemm_nn;; tn) K=gemm_tn;; spmm) K=spmm_kernel;; dense_nn) K=gemm_nn;; dense_tn) K=gemm_tn;; esac
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o $OUT/traffic_$M \
      python scripts/traffic_probe.py $M > $OUT/traffic_$M.json 2> $OUT/traffic_$M.err
done
timeout 1200 python -m pytest tests/test_gpu_fullsize_c3c4.py -q -x --timeout 900 > $OUT/c3c4_tests.log 2>&1
for C in C3 C4; do for A in lanczos rsvd; do
  timeout 900 python bench.py --config $C --algo $A --steps 2 --warmup 3 --e2e-steps 1 --cpu-budget 20 \
     > $OUT/bench_${C}_${A}.json 2> $OUT/bench_${C}_${A}.err
done; done
tail -3 $OUT/c3c4_tests.log
