#!/bin/bash
# gemm_nn warp-private epilogue (direct Z stores, per-warp symmetric Gram): parity, C2/C3/C5.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
timeout 300 python scripts/bench_kernels.py nn 2>&1 | tail -8
for CFG in C2 C3; do
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$CFG.json 2>gpurun_out/bench_$CFG.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$CFG.json').read().strip().splitlines()[-1])
print('$CFG TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy']['e_max'])
"
done
timeout -s ABRT 900 python -X faulthandler bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5b.json 2> gpurun_out/bench_C5b.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C5b.json').read().strip().splitlines()[-1])
print('C5', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['roofline']['frac'])
"
