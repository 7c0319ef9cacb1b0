#!/bin/bash
# Finaliser reduction with overlapped loads (w = 32): parity, C3/C4 lines, e2e breakdown.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_fullsize_c3c4.py -q -x 2>&1 | tail -1
for CFG in C3 C4; do
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$CFG.json 2>gpurun_out/bench_$CFG.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$CFG.json').read().strip().splitlines()[-1])
print('$CFG TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy']['e_max'])
"
done
timeout 300 python scripts/e2e_breakdown.py 2>&1 | tail -6
# (appended) short-row batch A/B
for SB in 8 4; do TSVD_SPMM_SB=$SB SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm 2>&1 | grep spmm | sed "s/^/SB=$SB /"; done
TSVD_SPMM_SB=4 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k spmm 2>&1 | tail -1
