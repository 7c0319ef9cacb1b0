#!/bin/bash
# the paper's dense workload (Sec. 4.2, Fig. 4) at its own sizes.
mkdir -p gpurun_out
timeout 1500 python scripts/fig4_dense.py > gpurun_out/fig4_dense.jsonl 2> gpurun_out/fig4_dense.err
echo "rc=$?"; tail -3 gpurun_out/fig4_dense.err | cut -c1-300
python -c "
import json
for ln in open('gpurun_out/fig4_dense.jsonl'):
    d=json.loads(ln); print(d['m'], d['algo'], d['paper_setting'], d['ms_median'], d['cycles'], '%.1e'%max(d['R']), '%.1e'%d['sigma_err_max'], '%.1e'%d['UtU_minus_I'])
"
# finaliser launch durations inside a C4 solve (which part of ortho_small is the kernel)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"finalize|prereduce" -c 60 --csv \
   --log-file gpurun_out/fin_c4.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/fin_c4.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ik,iv,iu=H.index('Kernel Name'),H.index('Metric Value'),H.index('Metric Unit')
import collections; agg=collections.defaultdict(list)
for r in rows[h+1:]:
    if len(r)>iv: agg[r[ik][:40]].append((float(r[iv].replace(',','')), r[iu]))
for k,v in agg.items(): print(k, len(v), v[:6])
PY
