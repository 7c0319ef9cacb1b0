#!/bin/bash
# SpMM 64-column launches for wide blocks: parity, RandSVD C3/C4 lines, C2 line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for A in "C3 rsvd" "C4 rsvd" "C2 lanczos"; do
  set -- $A
  timeout 900 python bench.py --config $1 --algo $2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$1_$2.json 2>gpurun_out/bench_$1_$2.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$1_$2.json').read().strip().splitlines()[-1])
print('$1 $2', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['accuracy']['e_max'])
"
done
