#!/bin/bash
# GPU session S3D: k_prefilter_cols tiling -- 8 rows per CTA, register caps for 6 / 8 CTAs per SM
O=gpurun_out/r2/s3d
mkdir -p $O
timeout 2000 python tools/ab.py 64 1 3 6 paper_2309_11072_b200/libhdll_b200.so exp/cr8/libhdll_b200.so exp/pfmb6/libhdll_b200.so exp/cr8mb8/libhdll_b200.so > $O/ab.log 2>&1; echo "ab rc=$?"; cat $O/ab.log
