#!/bin/bash
# GPU session AD: pairwise nodes on a side stream beside the ddot sweep, A/B c1 and c3 (+ parity of the experiment lib)
O=gpurun_out/r2
mkdir -p $O
HDLL_B200_LIB=$PWD/exp/nodeside/libhdll_b200.so timeout 900 python -m pytest tests/test_gpu_configs.py -q -x --timeout=600 -p no:cacheprovider -k "config1" > $O/gpu_tests_ad.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_ad.log
timeout 1200 python tools/ab.py 64 1 3 6 exp/head/libhdll_b200.so exp/nodeside/libhdll_b200.so > $O/ab_ad.log 2>&1; echo "ab rc=$?"; cat $O/ab_ad.log
timeout 1200 python tools/ab.py 1 3 3 6 exp/head/libhdll_b200.so exp/nodeside/libhdll_b200.so > $O/ab_ad3.log 2>&1; echo "ab c3 rc=$?"; cat $O/ab_ad3.log
