#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -x --timeout 600 -k "svd or lanczos or thick or c1 or rank or full" 2>&1 | tail -2
TSVD_LIB=ab_libs/libtsvd_jt.so python scripts/jac_timing.py 2>&1 | tail -7
SVD_D=28,128,200,384,450,640,704 timeout 600 python scripts/bench_kernels.py svd 2>&1
