# round-end rehearsal: full -m gpu suite, smoke, default bench line, reference arm,
# and the row-partitioned C5 harness path at world 1 (TSVD_BENCH_DIST=1)
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $O/s17_pytest.log 2>&1
echo pytest rc $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s17_smoke.log 2>&1
echo smoke rc $?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/s17_bench.json 2> $O/s17_bench.err
echo bench rc $?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/s17_ref.json 2> $O/s17_ref.err
echo ref rc $?
TSVD_BENCH_DIST=1 timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline > $O/s17_c5dist.json 2> $O/s17_c5dist.err
echo c5dist rc $?
echo done
