#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 600 > $OUT/kern_tests.log 2>&1
tail -3 $OUT/kern_tests.log
timeout 600 python scripts/bench_kernels.py dense > $OUT/kbench.log 2>&1
cat $OUT/kbench.log
timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
     > $OUT/bench_C4_lanczos.json 2> $OUT/bench_C4_lanczos.err
timeout 600 python bench.py --config C4 --algo rsvd --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
     > $OUT/bench_C4_rsvd.json 2> $OUT/bench_C4_rsvd.err
