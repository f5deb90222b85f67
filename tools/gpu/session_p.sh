#!/bin/bash
# GPU session P: plane coder count pass on SIMD words -- parity subset, then A/B against HEAD on c1 and c3
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout=600 -p no:cacheprovider -k "plane or golden or wide or config1 or config2" > $O/gpu_tests_p.log 2>&1; echo "tests rc=$?"; tail -3 $O/gpu_tests_p.log
timeout 900 python tools/ab.py 64 1 3 6 exp/head/libhdll_b200.so paper_2309_11072_b200/libhdll_b200.so > $O/ab_p_c1.log 2>&1; echo "ab c1 rc=$?"; cat $O/ab_p_c1.log
