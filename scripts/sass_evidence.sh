#!/bin/bash
# SASS instruction evidence per kernel of the built library (cuobjdump -sass):
# UTMALDG = TMA tensor loads (.2D, .2D.GATHER4), UBLKCP = 1-D bulk copies,
# DMMA = FP64 tensor-core mma.sync m8n8k4, SYNCS.* = mbarrier ops,
# ACQBULK / PREEXIT = griddepcontrol.wait / launch_dependents (PDL).
#   bash scripts/sass_evidence.sh > profiles/r02s/sass_evidence.txt
cd "$(dirname "$0")/.."
cuobjdump -sass paper_2403_06218_b200/libtsvd.so | awk '
/Function : /{ if (name != "") emit(); name=$3; delete c; next }
{ for (i = 1; i <= NF; i++) { t=$i; gsub(/;/, "", t);
    if (t ~ /^(UTMALDG|UBLKCP|DMMA|DFMA|LDGSTS|ACQBULK|PREEXIT|SYNCS\.ARRIVE\.TRANS64)/) { split(t, a, "."); k=a[1]; if (t ~ /GATHER4/) k=k".GATHER4"; c[k]++ } } }
function emit(  s, k) { s=""; for (k in c) s=s" "k"="c[k]; if (s != "") print name s }
END { if (name != "") emit() }' | c++filt | sed 's/(.*)//' | sort | uniq
