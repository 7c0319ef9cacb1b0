cd $GRAFT_REPO_ROOT
O=gpurun_out
for DK in "640 0" "384 128" "448 128" "512 128" "512 192"; do
set -- $DK
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --d $1 --keep $2 --maxit 12 > $O/s37_c3_d$1_k$2.json 2> $O/s37_c3_d$1_k$2.err
python -c "
import json; d=json.load(open('$O/s37_c3_d$1_k$2.json')); print('d=$1 keep=$2', d['value'], d['solver']['cycles'], d['solver']['nconv'], d['accuracy']['e_max'], d['clocks']['sm_mhz'])" >> $O/s37_sweep.log
done
echo done
