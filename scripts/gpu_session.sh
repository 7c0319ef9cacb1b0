set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_loopback.py tests/test_gpu_kernels.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > $O/s7_pytest.log 2>&1
echo pytest rc $?
SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm > $O/s7_spmm.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/s7_bench.json 2> $O/s7_bench.err
TSVD_GRAPHS=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/s7_bench_nograph.json 2> $O/s7_bench_nograph.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ortho bcgs_pip2 > $O/s7_bench_pip2.json 2> $O/s7_bench_pip2.err
echo done
