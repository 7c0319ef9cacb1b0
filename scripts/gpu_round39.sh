#!/bin/bash
# Jacobi configuration sweep at the solver sizes (d = 384 C2, 640 C3, 704 C4).
for JC in 4 8; do for NT in 128 256; do
  echo "== JC=$JC NT=$NT"
  TSVD_JACOBI_JC=$JC TSVD_JACOBI_NT=$NT SVD_D=384,640,704 timeout 300 python scripts/bench_kernels.py svd 2>&1 | tail -3
done; done
