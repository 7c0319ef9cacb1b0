#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
for KD in "640 320" "640 192" "512 256" "448 224"; do
  set -- $KD
  timeout 900 python bench.py --config C3 --d $1 --keep $2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
     > $OUT/bench_C3_thick_$1_$2.json 2> $OUT/bench_C3_thick_$1_$2.err
  python -c "
import json
d=json.loads(open('$OUT/bench_C3_thick_$1_$2.json').read().strip().splitlines()[-1])
print('d=$1 keep=$2 TTS %.4f'%d['value'], d['solver'], 'e_max %.1e'%d['accuracy']['e_max'])
"
done
