cd $GRAFT_REPO_ROOT
O=gpurun_out
for DK in "704 0" "448 224" "512 224" "576 256"; do
set -- $DK
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --d $1 --keep $2 --maxit 20 > $O/s38_c4_d$1_k$2.json 2> $O/s38_c4_d$1_k$2.err
python -c "
import json; d=json.load(open('$O/s38_c4_d$1_k$2.json')); print('d=$1 keep=$2', d['value'], d['solver']['cycles'], d['solver']['nconv'], d['accuracy']['e_max'], d['clocks']['sm_mhz'])" >> $O/s38_sweep.log
done
echo done
