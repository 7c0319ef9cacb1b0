cd $GRAFT_REPO_ROOT
O=gpurun_out
EQ_DSWEEP=1 timeout 1500 python scripts/equal_accuracy.py C3 C4 > $O/s34_dsweep.jsonl 2> $O/s34_dsweep.err
echo done
