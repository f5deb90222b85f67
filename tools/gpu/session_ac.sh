#!/bin/bash
# GPU session AC: S* tile window by TMA bulk copy in k_sort_scatter -- parity subset, A/B on c1 and c3
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tiled.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_ac.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_ac.log
timeout 1200 python tools/ab.py 64 1 3 6 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_ac.log 2>&1; echo "ab rc=$?"; cat $O/ab_ac.log
timeout 1200 python tools/ab.py 1 3 3 6 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_ac3.log 2>&1; echo "ab c3 rc=$?"; cat $O/ab_ac3.log
