set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
for F in 1 0; do
  TSVD_FOLD_S5=$F timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s21_bench_s5_$F.json 2> $O/s21_bench_s5_$F.err
done
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 900 > $O/s21_pytest.log 2>&1
echo pytest rc $?
echo done
