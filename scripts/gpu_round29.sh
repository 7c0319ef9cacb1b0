#!/bin/bash
# Rolled shared-memory Cholesky in the finaliser: parity, finaliser launch times, C2/C3/C4 lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"finalize|prereduce" -c 60 --csv \
   --log-file gpurun_out/fin_c4.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/fin_c4.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ik,iv,iu=H.index('Kernel Name'),H.index('Metric Value'),H.index('Metric Unit')
agg=collections.defaultdict(list)
for r in rows[h+1:]:
    if len(r)>iv: agg[r[ik][:40]].append(float(r[iv].replace(',','')))
for k,v in agg.items(): print(k, len(v), 'mean', sum(v)/len(v))
PY
for CFG in C2 C3 C4; do
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$CFG.json 2>gpurun_out/bench_$CFG.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$CFG.json').read().strip().splitlines()[-1])
print('$CFG TTS', d['value'], ' '.join('%s=%.2f'%(k,v['ms_per_step']) for k,v in d['phases'].items()), d['e2e']['value'], d['roofline']['frac'], d['accuracy']['e_max'])
"
done
