#!/bin/bash
# SpMM A/B: 8 lanes x 2 columns (default) vs 4 lanes x 4 columns (TSVD_SPMM_V4=1: 8-nz, 2: 4-nz batches).
mkdir -p gpurun_out
for V in 0 1 2; do TSVD_SPMM_V4=$V SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm 2>&1 | grep spmm | sed "s/^/V4=$V /"; done
for V in 1 2; do TSVD_SPMM_V4=$V timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k spmm 2>&1 | tail -1; done
