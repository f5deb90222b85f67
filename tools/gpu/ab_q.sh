#!/bin/bash
# A/B of experiment libraries on c1 (64 images): tools/gpu/ab_q.sh TAG LIB...
O=gpurun_out/r2
mkdir -p $O
T=$1; shift
timeout 1200 python tools/ab.py 64 1 3 6 "$@" > $O/ab_$T.log 2>&1; echo "ab rc=$?"; cat $O/ab_$T.log
