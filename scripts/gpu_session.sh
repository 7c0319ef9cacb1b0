cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 > $O/s13_bench_C2.json 2> $O/s13_bench_C2.err
timeout 600 python -m pytest tests/test_gpu_solvers.py -x -q -p no:cacheprovider -k "c1 or inplace" > $O/s13_pytest.log 2>&1
echo "pytest rc $?" >> $O/s13_pytest.log
echo done
