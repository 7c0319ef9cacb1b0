cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "tn or cgs or chol" > $O/s17_pytest.log 2>&1
echo "pytest rc $?" >> $O/s17_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s17_bench_C2.json 2> $O/s17_bench_C2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/s17_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
echo done
