#!/bin/bash
# Pipelined short-row SpMM: parity in every mode, A/B timing, C2 bench.
mkdir -p gpurun_out
for P in 1 2; do TSVD_SPMM_PIPE=$P timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "spmm" 2>&1 | tail -1; done
for P in 0 1 2; do TSVD_SPMM_PIPE=$P SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm 2>&1 | grep spmm; done
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C2.json').read().strip().splitlines()[-1])
print('C2 TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy']['e_max'])
"
