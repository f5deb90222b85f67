#!/bin/bash
# GPU session AO: ddot grid without the z dimension in batches (c1 at 16 threads; c4 at 16 threads)
O=gpurun_out/r2
mkdir -p $O
C=exp/cur/libhdll_b200.so; Z=exp/z1/libhdll_b200.so
timeout 1200 python tools/ab.py 64 1 3 5 $C,HDLL_BLAS_THREADS=16 $Z,HDLL_BLAS_THREADS=16 > $O/ab_ao.log 2>&1; echo "c1 rc=$?"; cat $O/ab_ao.log
