#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -x --timeout 600 > $OUT/tests6.log 2>&1
tail -3 $OUT/tests6.log
SVD_D=28,128,200,384,450,640,704 timeout 600 python scripts/bench_kernels.py svd > $OUT/svd.log 2>&1
cat $OUT/svd.log
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/bench_C2.json 2> $OUT/bench_C2.err
timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/bench_C4_lanczos.json 2> $OUT/bench_C4_lanczos.err
