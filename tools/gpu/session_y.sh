#!/bin/bash
# GPU session Y: parity subset on the shipped library, A/B (HEAD vs current) on c1
O=gpurun_out/r2
mkdir -p $O
T=${TAG:-y}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_plugin.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_$T.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests_$T.log
timeout 1200 python tools/ab.py 64 1 3 6 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_$T.log 2>&1; echo "ab rc=$?"; cat $O/ab_$T.log
