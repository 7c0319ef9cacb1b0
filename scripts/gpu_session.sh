# one gpurun session (development)
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_loopback.py -m gpu -q -p no:cacheprovider > $O/s4_loop.log 2>&1
echo loop rc $?
for S in 0 1; do
  TSVD_SPMM_STAGED=$S SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm > $O/s4_spmm_$S.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider > $O/s4_pytest.log 2>&1
echo pytest rc $?
SPMM_CFG=C2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmm_staged -s 2 -c 1 -o $O/s4_spmm_staged python scripts/bench_kernels.py spmm > $O/s4_ncu.log 2>&1
timeout 300 python scripts/e2e_breakdown.py > $O/s4_e2e.log 2>&1
echo done
