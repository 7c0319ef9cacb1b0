set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
./scripts/l2probe.bin > $O/s5_l2probe.log 2>&1
for S in 0 1; do
  TSVD_SPMM_STAGED=$S SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm > $O/s5_spmm_$S.log 2>&1
done
SPMM_CFG=C2 TSVD_SPMM_STAGED=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmm_kernel -s 2 -c 1 -o $O/s5_spmm_old python scripts/bench_kernels.py spmm > $O/s5_ncu_old.log 2>&1
SPMM_CFG=C2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmm_staged -s 2 -c 1 -o $O/s5_spmm_staged python scripts/bench_kernels.py spmm > $O/s5_ncu.log 2>&1
echo done
