# round-2 evidence: C2 launch list, full capture of the top kernels, traffic of the benched launches
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02_C2_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_nn_tma_kernel --csv --log-file $O/r02_traffic_ortho_nn.csv $B > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tn_tma_kernel --csv --log-file $O/r02_traffic_ortho_tn.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_nn_tma_kernel -s 60 -c 2 -o $O/r02_full_nn $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tn_tma_kernel -s 60 -c 1 -o $O/r02_full_tn $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_kernel -s 20 -c 1 -o $O/r02_full_spmm $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_reg_kernel -c 1 -o $O/r02_full_jacobi $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rowT_kernel -s 40 -c 1 -o $O/r02_full_rowt $B > /dev/null 2>&1
echo done
