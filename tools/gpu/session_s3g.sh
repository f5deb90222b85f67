#!/bin/bash
# GPU session S3G: k_sdr_ycc's four pixels as one straight-line block (A/B + parity)
O=gpurun_out/r2/s3g
mkdir -p $O
timeout 1500 python tools/ab.py 64 1 3 6 paper_2309_11072_b200/libhdll_b200.so exp/sdrilp/libhdll_b200.so > $O/ab.log 2>&1; echo "ab rc=$?"; cat $O/ab.log
HDLL_B200_LIB=$PWD/exp/sdrilp/libhdll_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
