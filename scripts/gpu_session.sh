# round-2 evidence: C2 launch list, full capture of the top kernels (exported
# to CSV on the box: the .ncu-rep files are too large to bring back), traffic
# of the benched launches
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out
T=/tmp/ncu_r02
mkdir -p $T
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02_C2_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_nn_tma_kernel --csv --log-file $O/r02_traffic_ortho_nn.csv $B > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tn_tma_kernel --csv --log-file $O/r02_traffic_ortho_tn.csv $B > /dev/null 2>&1
for K in "gemm_nn_tma_kernel:60:2" "gemm_tn_tma_kernel:60:1" "spmm_kernel:20:1" "jacobi_reg_kernel:0:1" "rowT_kernel:40:1"; do
  N=${K%%:*}; R=${K#*:}; S=${R%%:*}; C=${R##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$N -s $S -c $C -o $T/full_$N $B > /dev/null 2>&1
  ncu -i $T/full_$N.ncu-rep --page raw --csv > $O/r02_full_${N}_raw.csv 2>/dev/null
  ncu -i $T/full_$N.ncu-rep --page details --csv > $O/r02_full_${N}_details.csv 2>/dev/null
done
ncu -i $T/full_gemm_nn_tma_kernel.ncu-rep --page source --csv --print-source sass > $O/r02_full_nn_sass.csv 2>/dev/null
du -sh $O
echo done
