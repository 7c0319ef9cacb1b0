#!/bin/bash
# In-place outputs, SpMM column-slice A/B, first C5 run (1e9 nnz on one GPU).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv | tail -1
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/c5_mem.log; sleep 2; done ) &
MP=$!
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
kill $MP
tail -5 gpurun_out/bench_C5.err | cut -c1-400

sort -n gpurun_out/c5_mem.log | tail -1
python -c "
import json
d=json.loads(open('gpurun_out/bench_C5.json').read().strip().splitlines()[-1])
print('C5', d['value'], d['solver'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['roofline'])
"
