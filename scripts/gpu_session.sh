cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solvers.py -x -q -p no:cacheprovider > $O/s21_pytest.log 2>&1
echo "pytest rc $?" >> $O/s21_pytest.log
for V in 0 1; do
TSVD_SVD_OVERLAP=$V timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s21_bench_C2_ov$V.json 2> $O/s21_bench_C2_ov$V.err
TSVD_SVD_OVERLAP=$V timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s21_bench_C4_ov$V.json 2> $O/s21_bench_C4_ov$V.err
done
for V in 0 1; do
TSVD_SVD_OVERLAP=$V timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s21_bench_C2b_ov$V.json 2> $O/s21_bench_C2b_ov$V.err
done
echo done
