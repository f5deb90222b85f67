#!/bin/bash
# GPU session S3C: k_sdr_ycc variants -- fp32 magic floor, bit-built RGBE floats, fewer registers (5 / 6 CTAs per SM)
O=gpurun_out/r2/s3c
mkdir -p $O
timeout 2000 python tools/ab.py 64 1 3 6 paper_2309_11072_b200/libhdll_b200.so exp/ffloor/libhdll_b200.so exp/fbits/libhdll_b200.so exp/fboth/libhdll_b200.so exp/sdr5/libhdll_b200.so exp/sdr6/libhdll_b200.so > $O/ab.log 2>&1; echo "ab rc=$?"; cat $O/ab.log
