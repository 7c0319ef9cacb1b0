cd $GRAFT_REPO_ROOT
O=gpurun_out
for DK in "384 0" "192 64" "256 64" "256 128" "320 64" "320 128"; do
set -- $DK
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --d $1 --keep $2 --maxit 12 > $O/s36_c2_d$1_k$2.json 2> $O/s36_c2_d$1_k$2.err
python -c "
import json; d=json.load(open('$O/s36_c2_d$1_k$2.json')); print('d=$1 keep=$2', d['value'], d['solver']['cycles'], d['solver']['nconv'], d['accuracy']['e_max'], d['clocks']['sm_mhz'])" >> $O/s36_sweep.log
done
echo done
