#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
for L in "" ab_libs/libtsvd_pf6.so ab_libs/libtsvd_pf8.so; do
  echo "== lib $L"
  TSVD_LIB=$L timeout 300 python scripts/bench_kernels.py nn 2>&1 | grep "s=0"
done > $OUT/rowt_ab.log 2>&1
cat $OUT/rowt_ab.log
for JC in 2 4 8; do
  echo "== JC $JC"
  TSVD_JACOBI_JC=$JC SVD_D=128,384,704 timeout 300 python scripts/bench_kernels.py svd 2>&1
done > $OUT/jac_ab.log 2>&1
cat $OUT/jac_ab.log
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x > $OUT/dist.log 2>&1; tail -2 $OUT/dist.log
