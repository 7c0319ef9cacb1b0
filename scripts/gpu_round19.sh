#!/bin/bash
# C5 on one GPU (1e9 nonzeros, d = 160), with progress logging and a traceback on timeout.
mkdir -p gpurun_out
TSVD_GEN_VERBOSE=1 timeout -s ABRT 900 python -X faulthandler bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
echo "rc=$?"
grep -v "^ *$" gpurun_out/bench_C5.err | tail -40 | cut -c1-300
python -c "
import json
d=json.loads(open('gpurun_out/bench_C5.json').read().strip().splitlines()[-1])
print('C5', d['value'], d['solver'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['roofline'])
"
