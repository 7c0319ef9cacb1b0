#!/bin/bash
# Multi-CTA Gram pre-reduction (w >= 23): full GPU suite, C2/C3/C4 lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for CFG in C2 C3 C4; do
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$CFG.json 2>gpurun_out/bench_$CFG.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$CFG.json').read().strip().splitlines()[-1])
print('$CFG TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy']['e_max'])
"
done
