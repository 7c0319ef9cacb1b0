#!/bin/bash
for NT in 0 128; do
  echo "== NT $NT"
  TSVD_JACOBI_NT=$NT SVD_D=28,128,200,384,450,704 timeout 600 python scripts/bench_kernels.py svd 2>&1
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C2.json').read().strip().splitlines()[-1])
print('C2 TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'])
"
