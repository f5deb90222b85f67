#!/bin/bash
# GPU session U: fast serial decoder -- decode tests, then decode timing new vs HEAD
O=gpurun_out/r2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x --timeout=300 -p no:cacheprovider > $O/dec_tests_u.log 2>&1; echo "dec tests rc=$?"; tail -15 $O/dec_tests_u.log
HDLL_B200_LIB=$PWD/exp/head/libhdll_b200.so timeout 600 python -m pytest tests/test_gpu_decode.py -q -x --timeout=300 -p no:cacheprovider -k truncated > $O/dec_tests_u_head.log 2>&1; echo "head robust rc=$?"; tail -5 $O/dec_tests_u_head.log
timeout 300 python tools/decode_time.py 64 > $O/dec_time_u.log 2>&1; echo "new rc=$?"; tail -2 $O/dec_time_u.log
HDLL_B200_LIB=$PWD/exp/head/libhdll_b200.so timeout 300 python tools/decode_time.py 64 > $O/dec_time_u_head.log 2>&1; echo "head rc=$?"; tail -2 $O/dec_time_u_head.log
