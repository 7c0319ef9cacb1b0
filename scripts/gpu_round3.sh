#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/gpu_tests.log 2>&1
tail -3 $OUT/gpu_tests.log
timeout 600 python scripts/c3_debug.py 0.1 32 640 1 > $OUT/c3dbg.log 2>&1
timeout 600 python scripts/c3_debug.py 1.0 32 640 1 >> $OUT/c3dbg.log 2>&1
for KD in "160 64" "192 64" "224 80" "256 96" "128 64"; do
  set -- $KD
  timeout 600 python bench.py --config C2 --d $1 --keep $2 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
     > $OUT/bench_C2_thick_$1_$2.json 2> $OUT/bench_C2_thick_$1_$2.err
done
for C in C3 C4; do
  timeout 900 python bench.py --config $C --steps 2 --warmup 3 --e2e-steps 1 --cpu-budget 20 \
     > $OUT/bench_${C}_lanczos.json 2> $OUT/bench_${C}_lanczos.err
done
