#!/bin/bash
# GPU session AG: deep-pipeline ddot for big segments -- parity subset, A/B c1, c3, c2
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tiled.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_ag.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_ag.log
timeout 1200 python tools/ab.py 1 3 3 6 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_ag3.log 2>&1; echo "ab c3 rc=$?"; cat $O/ab_ag3.log
timeout 1200 python tools/ab.py 1 2 3 6 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_ag2.log 2>&1; echo "ab c2 rc=$?"; cat $O/ab_ag2.log
timeout 1200 python tools/ab.py 64 1 3 6 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_ag.log 2>&1; echo "ab c1 rc=$?"; cat $O/ab_ag.log
