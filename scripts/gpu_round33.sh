#!/bin/bash
# Evidence refresh after the gemm_nn epilogue change: official C2 line + ref arm + ncu (round26),
# C5 line with the host-oracle sample, C4 line.
bash scripts/gpu_round26.sh
timeout -s ABRT 1200 python -X faulthandler bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
for CFG in C5 C4 C3; do python -c "
import json
d=json.loads(open('gpurun_out/bench_$CFG.json').read().strip().splitlines()[-1])
print('$CFG', d['value'], d['solver']['cycles'], d['roofline']['kernel'], d['roofline']['frac'], (d.get('cpu_baseline') or {}).get('value'))
"; done
du -sh gpurun_out
