#!/bin/bash
# Row-sorted CSR layout: parity, SpMM timing, ncu capture of the C2 product, C2 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm 2>&1 | grep spmm
SPMM_CFG=C2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmm_kernel -s 3 -c 1 \
   -o gpurun_out/spmm_c2_sorted python scripts/bench_kernels.py spmm > gpurun_out/ncu_spmm.log 2>&1
tail -2 gpurun_out/ncu_spmm.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C2.json').read().strip().splitlines()[-1])
print('C2 TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy'])
"
