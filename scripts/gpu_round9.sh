#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/tests9.log 2>&1
tail -3 $OUT/tests9.log
timeout 600 python scripts/e2e_breakdown.py > $OUT/e2e.log 2>&1
cat $OUT/e2e.log
timeout 900 python bench.py > $OUT/bench_C2.json 2> $OUT/bench_C2.err
tail -c 600 $OUT/bench_C2.json
