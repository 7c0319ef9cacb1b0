#!/bin/bash
# Finaliser reduction with overlapped loads (w = 32): parity, C3/C4 lines, e2e breakdown.
mkdir -p gpurun_out
# (appended) short-row batch A/B
for SB in 8 4; do TSVD_SPMM_SB=$SB SPMM_CFG=C2,C3 timeout 300 python scripts/bench_kernels.py spmm 2>&1 | grep spmm | sed "s/^/SB=$SB /"; done
TSVD_SPMM_SB=4 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k spmm 2>&1 | tail -1
