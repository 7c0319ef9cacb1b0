cd $GRAFT_REPO_ROOT
O=gpurun_out
for V in 1 0 1; do
TSVD_SVD_OVERLAP=$V timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 > $O/s28_e2e_ov$V.json 2> $O/s28_e2e_ov$V.err
python -c "
import json; d=json.load(open('$O/s28_e2e_ov$V.json')); print('ov$V', d['value'], d['e2e']['value'], d['e2e']['steps_ms_create_solve_get_destroy'])" >> $O/s28_e2e.log
done
timeout 900 python -m pytest tests/test_gpu_solvers.py -x -q -p no:cacheprovider > $O/s28_pytest.log 2>&1
echo "pytest rc $?" >> $O/s28_pytest.log
echo done
