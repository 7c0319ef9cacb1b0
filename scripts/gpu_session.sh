cd $GRAFT_REPO_ROOT
O=gpurun_out
for G in 1 0 1 0; do
TSVD_GET_2STREAM=$G timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 8 > $O/s30_e2e_g$G.json 2> $O/s30_e2e_g$G.err
python -c "
import json; d=json.load(open('$O/s30_e2e_g$G.json')); print('g$G', d['e2e']['value'], d['e2e']['steps_ms_create_solve_get_destroy'])" >> $O/s30_e2e.log
done
echo done
