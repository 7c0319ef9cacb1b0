#!/bin/bash
# N4 threshold driver + finaliser (register w <= 16 / rolled w = 32): parity, C2 line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C2.json').read().strip().splitlines()[-1])
print('C2 TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy']['e_max'])
"
