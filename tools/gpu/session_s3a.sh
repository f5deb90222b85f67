#!/bin/bash
# GPU session S3A: two-stream co-scheduling diagnostic; fp64 quantiser by certified reciprocal (A/B + parity)
O=gpurun_out/r2/s3a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 600 python tools/concurrency.py 64 2 > $O/conc2.log 2>&1; echo "conc2 rc=$?"; cat $O/conc2.log | tail -4
timeout 600 python tools/concurrency.py 64 4 > $O/conc4.log 2>&1; echo "conc4 rc=$?"; cat $O/conc4.log | tail -4
HDLL_B200_LIB=$PWD/exp/qrcp/libhdll_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider > $O/qrcp_tests.log 2>&1; echo "qrcp tests rc=$?"; tail -2 $O/qrcp_tests.log
timeout 1200 python tools/ab.py 64 1 3 6 paper_2309_11072_b200/libhdll_b200.so exp/qrcp/libhdll_b200.so > $O/ab_qrcp.log 2>&1; echo "ab rc=$?"; cat $O/ab_qrcp.log
