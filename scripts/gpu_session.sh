cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 900 > $O/s31_pytest.log 2>&1
echo "pytest rc $?" >> $O/s31_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s31_smoke.log 2>&1
timeout 900 python bench.py > $O/s31_bench_default.json 2> $O/s31_bench_default.err
echo done
