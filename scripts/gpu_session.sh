set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python tests/c5g2_check.py > $O/s8_c5g2.json 2> $O/s8_c5g2.err
echo c5g2 rc $?
timeout 1500 python bench.py --config C5g2 --steps 1 --warmup 1 --no-cpu-baseline > $O/s8_bench_c5g2.json 2> $O/s8_bench_c5g2.err
echo bench c5g2 rc $?
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline > $O/s8_bench_c5.json 2> $O/s8_bench_c5.err
echo bench c5 rc $?
echo done
