#!/bin/bash
# GPU session AK: ddot staging block size at the 16-thread and 1-thread parity models, c1 and c3
O=gpurun_out/r2
mkdir -p $O
L="exp/cur/libhdll_b200.so exp/b512/libhdll_b200.so exp/b1024/libhdll_b200.so exp/b1024s2/libhdll_b200.so"
A16=""; for l in $L; do A16="$A16 $l,HDLL_BLAS_THREADS=16"; done
timeout 1500 python tools/ab.py 64 1 2 5 $A16 > $O/ab_ak16.log 2>&1; echo "c1 t16 rc=$?"; cat $O/ab_ak16.log
timeout 1500 python tools/ab.py 64 1 2 5 $L > $O/ab_ak1.log 2>&1; echo "c1 t1 rc=$?"; cat $O/ab_ak1.log
timeout 1500 python tools/ab.py 1 3 2 5 $A16 > $O/ab_ak316.log 2>&1; echo "c3 t16 rc=$?"; cat $O/ab_ak316.log
