#!/bin/bash
# GPU session K: DCT coder blocks per lane (1, 2, 4): parity, then A/B on c1 and c3
O=gpurun_out/r2
mkdir -p $O
for b in 2 4; do
  HDLL_B200_LIB=$PWD/exp/bpl$b/libhdll_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout=600 -p no:cacheprovider -k "golden or c1 or c3" > $O/gpu_tests_bpl$b.log 2>&1; echo "bpl$b tests rc=$?"; tail -1 $O/gpu_tests_bpl$b.log
done
timeout 900 python tools/ab.py 64 1 3 6 exp/base/libhdll_b200.so exp/bpl1/libhdll_b200.so exp/bpl2/libhdll_b200.so exp/bpl4/libhdll_b200.so > $O/ab_bpl_c1.log 2>&1; echo "ab c1 rc=$?"; cat $O/ab_bpl_c1.log
timeout 900 python tools/ab.py 1 3 3 6 exp/bpl1/libhdll_b200.so exp/bpl2/libhdll_b200.so exp/bpl4/libhdll_b200.so > $O/ab_bpl_c3.log 2>&1; echo "ab c3 rc=$?"; cat $O/ab_bpl_c3.log
