cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_solvers.py -x -q -p no:cacheprovider -k "profiling_mask or c1_lanczos" > $O/s40_pytest.log 2>&1
echo "pytest rc $?" >> $O/s40_pytest.log
echo done
