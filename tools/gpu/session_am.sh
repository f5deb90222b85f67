#!/bin/bash
# GPU session AM: continuous ddot pipeline across chunks -- parity subset, A/B c1 (1 and 16 threads), c3 (16)
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tiled.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_am.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_am.log
H=exp/head/libhdll_b200.so; C=exp/cur/libhdll_b200.so
timeout 1200 python tools/ab.py 64 1 3 5 $H,HDLL_BLAS_THREADS=16 $C,HDLL_BLAS_THREADS=16 $H $C > $O/ab_am.log 2>&1; echo "c1 rc=$?"; cat $O/ab_am.log
timeout 1200 python tools/ab.py 1 3 3 5 $H,HDLL_BLAS_THREADS=16 $C,HDLL_BLAS_THREADS=16 > $O/ab_am3.log 2>&1; echo "c3 rc=$?"; cat $O/ab_am3.log
timeout 900 python bench.py --no-decode --no-cpu --steps 5 > $O/bench_am.log 2>&1; echo "bench rc=$?"; grep -o '"parity_vs_oracle": [^}]*}\|"value": [0-9.]*, "unit"' $O/bench_am.log | head -3
timeout 900 python bench.py --no-decode --steps 5 > $O/bench_am2.log 2>&1; echo "bench2 rc=$?"; grep -o '"parity_vs_oracle": [^}]*}' $O/bench_am2.log | head -3
