#!/bin/bash
# rowT symmetric Gram: parity, C2 / C5 lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C2.json').read().strip().splitlines()[-1])
print('C2 TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy']['e_max'])
"
timeout -s ABRT 900 python -X faulthandler bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5b.json 2> gpurun_out/bench_C5b.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C5b.json').read().strip().splitlines()[-1])
print('C5', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['roofline']['frac'])
"
