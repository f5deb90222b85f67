#!/bin/bash
# GPU session AB_PF: prefilter index arithmetic.  shipped = reflect_idx without the 64-bit division when one reflection suffices;
# exp/reflect64 = the old 64-bit modulo; exp/pfunroll = shipped + the horizontal pass of a full tile unrolled.  Parity tests first.
O=gpurun_out/r2/ab_pf
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tiled.py -m gpu -q -x -p no:cacheprovider > $O/tests_shipped.log 2>&1; echo "tests shipped rc=$?"; tail -1 $O/tests_shipped.log
HDLL_B200_LIB=$PWD/exp/pfunroll/libhdll_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $O/tests_pfunroll.log 2>&1; echo "tests pfunroll rc=$?"; tail -1 $O/tests_pfunroll.log
python tools/ab.py 64 1 4 6 paper_2309_11072_b200/libhdll_b200.so exp/reflect64/libhdll_b200.so exp/pfunroll/libhdll_b200.so > $O/ab_c1.txt 2>&1; cat $O/ab_c1.txt
python tools/ab.py 1 3 3 6 paper_2309_11072_b200/libhdll_b200.so exp/reflect64/libhdll_b200.so exp/pfunroll/libhdll_b200.so > $O/ab_c3.txt 2>&1; cat $O/ab_c3.txt
