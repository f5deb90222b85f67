#!/bin/bash
# GPU session L: DCT coder 4 vs 8 blocks per lane (max 8: more shared memory) on c1, c3, c2
O=gpurun_out/r2
mkdir -p $O
HDLL_B200_LIB=$PWD/exp/m8bpl8/libhdll_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -p no:cacheprovider -k "golden or wide" > $O/gpu_tests_bpl8.log 2>&1; echo "bpl8 tests rc=$?"; tail -1 $O/gpu_tests_bpl8.log
timeout 900 python tools/ab.py 64 1 3 6 exp/bpl4/libhdll_b200.so exp/m8bpl4/libhdll_b200.so exp/m8bpl8/libhdll_b200.so > $O/ab_bpl8_c1.log 2>&1; echo "ab c1 rc=$?"; cat $O/ab_bpl8_c1.log
timeout 900 python tools/ab.py 1 3 3 6 exp/bpl4/libhdll_b200.so exp/m8bpl8/libhdll_b200.so > $O/ab_bpl8_c3.log 2>&1; echo "ab c3 rc=$?"; cat $O/ab_bpl8_c3.log
timeout 900 python tools/ab.py 1 2 3 6 exp/bpl1/libhdll_b200.so exp/bpl4/libhdll_b200.so exp/m8bpl8/libhdll_b200.so > $O/ab_bpl8_c2.log 2>&1; echo "ab c2 rc=$?"; cat $O/ab_bpl8_c2.log
