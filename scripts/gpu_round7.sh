#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 600 -k spmm > $OUT/tests7.log 2>&1
tail -3 $OUT/tests7.log
timeout 600 python scripts/bench_kernels.py spmm > $OUT/spmm.log 2>&1
cat $OUT/spmm.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:spmm_kernel -c 1 -o $OUT/traffic_spmm \
    python scripts/traffic_probe.py spmm > $OUT/traffic_spmm.json 2> $OUT/traffic_spmm.err
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/bench_C2_$i.json 2> $OUT/bench_C2_$i.err
done
