#!/bin/bash
# GPU session AN: continuous ddot pipeline with the batch-size rule -- parity subset, A/B c1 and c3 at 16 threads
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tiled.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_an.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_an.log
H=exp/head/libhdll_b200.so; C=exp/cur/libhdll_b200.so
timeout 1200 python tools/ab.py 64 1 3 5 $H,HDLL_BLAS_THREADS=16 $C,HDLL_BLAS_THREADS=16 > $O/ab_an.log 2>&1; echo "c1 rc=$?"; cat $O/ab_an.log
timeout 1200 python tools/ab.py 1 3 3 5 $H,HDLL_BLAS_THREADS=16 $C,HDLL_BLAS_THREADS=16 > $O/ab_an3.log 2>&1; echo "c3 rc=$?"; cat $O/ab_an3.log
