set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider > $O/s15_pytest.log 2>&1
echo pytest rc $?
timeout 300 python scripts/bench_kernels.py nn32 nn > $O/s15_nn.log 2>&1
timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/s15_bench_C3.json 2> $O/s15_bench_C3.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_nn_tma_kernel -s 120 -c 1 -o $O/s15_nn32 python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $O/s15_ncu_nn.log 2>&1
timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/s15_bench_C4.json 2> $O/s15_bench_C4.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s15_bench.json 2> $O/s15_bench.err
echo done
