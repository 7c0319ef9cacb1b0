cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > $O/s14_pytest.log 2>&1
echo "pytest rc $?" >> $O/s14_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 > $O/s14_bench_C2.json 2> $O/s14_bench_C2.err
echo done
