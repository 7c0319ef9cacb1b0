#!/bin/bash
for NT in 256 128; do
  echo "== NT $NT"
  TSVD_JACOBI_NT=$NT SVD_D=28,128,384,704 timeout 600 python scripts/bench_kernels.py svd 2>&1
done
TSVD_JACOBI_NT=128 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k svd 2>&1 | tail -2
