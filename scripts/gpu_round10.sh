#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -x --timeout 600 > $OUT/tests10.log 2>&1
tail -3 $OUT/tests10.log
for v in 0 1; do TSVD_ROWT32=$v timeout 300 python scripts/bench_kernels.py nn 2>&1 | grep "s=0"; done
for C in C3 C4; do
  timeout 900 python bench.py --config $C --steps 2 --warmup 3 --e2e-steps 3 --cpu-budget 20 \
     > $OUT/bench_${C}_lanczos.json 2> $OUT/bench_${C}_lanczos.err
done
