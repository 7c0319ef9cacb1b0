cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1800 python scripts/fig4_dense.py > $O/s35_fig4.jsonl 2> $O/s35_fig4.err
echo done
