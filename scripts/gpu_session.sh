cd $GRAFT_REPO_ROOT
O=gpurun_out
for OR in cgs_cqr2 bcgs_pip2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --ortho $OR > $O/s39_c2_$OR.json 2> $O/s39_c2_$OR.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --ortho $OR --d 256 --keep 128 --maxit 12 > $O/s39_c2_thick_$OR.json 2> $O/s39_c2_thick_$OR.err
done
for f in $O/s39_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d['value'], d['solver']['cycles'], d['solver']['nconv'], d['solver']['breakdowns'], d['accuracy']['e_max'], d['clocks']['sm_mhz'])" >> $O/s39.log; done
echo done
