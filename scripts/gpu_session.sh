set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > $O/s9_pytest.log 2>&1
echo pytest rc $?
timeout 1200 python scripts/equal_accuracy.py C3 C4 > $O/s9_equal_accuracy.jsonl 2> $O/s9_equal_accuracy.err
echo eq rc $?
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > $O/s9_bench_C3.json 2> $O/s9_bench_C3.err
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/s9_bench_C4.json 2> $O/s9_bench_C4.err
echo done
