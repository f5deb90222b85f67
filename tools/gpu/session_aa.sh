#!/bin/bash
# GPU session AA: pairwise nodes fused into the ddot kernel -- parity subset, A/B on c1 and c3
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tiled.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_aa.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_aa.log
timeout 1200 python tools/ab.py 64 1 3 6 exp/sepnodes/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_aa.log 2>&1; echo "ab rc=$?"; cat $O/ab_aa.log
timeout 1200 python tools/ab.py 1 3 3 6 exp/sepnodes/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_aa3.log 2>&1; echo "ab c3 rc=$?"; cat $O/ab_aa3.log
