#!/bin/bash
# e2e re-check (C2) + breakdown
mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_C2.json').read().strip().splitlines()[-1])
print('C2 TTS', d['value'], d['e2e']['value'], d['roofline']['frac'])
"
done
timeout 300 python scripts/e2e_breakdown.py 2>&1 | tail -6
