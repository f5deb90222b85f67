#!/bin/bash
# GPU session AI: certified fp32 forward DCT variants, A/B on c1 (64 images)
O=gpurun_out/r2
mkdir -p $O
timeout 1500 python tools/ab.py 64 1 3 5 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so exp/nofb/libhdll_b200.so exp/rcpa/libhdll_b200.so exp/rcpanofb/libhdll_b200.so > $O/ab_ai.log 2>&1; echo "ab rc=$?"; cat $O/ab_ai.log
