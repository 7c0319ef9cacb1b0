set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
nvidia-smi --query-gpu=index,name,memory.used,utilization.gpu --format=csv > $O/s16_smi.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_loopback.py -m gpu -q -x -p no:cacheprovider --timeout 120 > $O/s16_pytest.log 2>&1
echo pytest rc $?
timeout 120 python scripts/bench_kernels.py nn32 nn > $O/s16_nn.log 2>&1
timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/s16_bench_C3.json 2> $O/s16_bench_C3.err
timeout 300 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/s16_bench_C4.json 2> $O/s16_bench_C4.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/s16_bench.json 2> $O/s16_bench.err
echo done
