cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py tests/test_gpu_n3_dense.py -x -q -p no:cacheprovider > $O/s16_pytest.log 2>&1
echo "pytest rc $?" >> $O/s16_pytest.log
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s16_bench_C4.json 2> $O/s16_bench_C4.err
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s16_bench_C3.json 2> $O/s16_bench_C3.err
timeout 1200 python bench.py --config C5g2 --steps 2 --warmup 3 --no-cpu-baseline > $O/s16_bench_C5g2.json 2> $O/s16_bench_C5g2.err
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $O/s16_bench_C5.json 2> $O/s16_bench_C5.err
echo done
