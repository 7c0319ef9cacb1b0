cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > $O/s23_pytest.log 2>&1
echo "pytest rc $?" >> $O/s23_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s23_bench_C2.json 2> $O/s23_bench_C2.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s23_bench_C4.json 2> $O/s23_bench_C4.err
echo done
