cd $GRAFT_REPO_ROOT
O=gpurun_out
for JC in 4 8; do for TOP in 0 100; do
echo "== JC $JC TOP $TOP"
TSVD_DBG_SVD_TOP=$TOP TSVD_JACOBI_JC=$JC TSVD_LIB=ab_libs/libtsvd_jt.so timeout 120 python scripts/jac_timing.py
done; done > $O/s3_jt.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -x -q -p no:cacheprovider > $O/s3_pytest.log 2>&1
echo "pytest rc $?" >> $O/s3_pytest.log
for R in 0 1; do
TSVD_ROWT_TMA=$R timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s3_bench_C2_rowt$R.json 2> $O/s3_bench_C2_rowt$R.err
TSVD_ROWT_TMA=$R timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s3_bench_C3_rowt$R.json 2> $O/s3_bench_C3_rowt$R.err
done
echo done
