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
