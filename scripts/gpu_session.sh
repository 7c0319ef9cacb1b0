cd $GRAFT_REPO_ROOT
O=gpurun_out
for M in all dominant none; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --prof-mode $M > $O/s6_bench_C2_$M.json 2> $O/s6_bench_C2_$M.err
done
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --prof-mode all > $O/s6_bench_C4_all.json 2> $O/s6_bench_C4_all.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/s6_bench_C4_dominant.json 2> $O/s6_bench_C4_dominant.err
echo done
