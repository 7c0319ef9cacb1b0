set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python scripts/bench_kernels.py nn32 nn > $O/s13_nn.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider > $O/s13_pytest.log 2>&1
echo pytest rc $?
timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/s13_bench_C3.json 2> $O/s13_bench_C3.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/s13_bench.json 2> $O/s13_bench.err
echo done
