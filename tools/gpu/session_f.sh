#!/bin/bash
# GPU session F (round 2): A/B (DCT coder coefficient prefetch + sort-scatter RGBE preload), band_begin steps
O=gpurun_out/r2
mkdir -p $O
timeout 900 python tools/ab.py 64 1 3 6 exp/base/libhdll_b200.so exp/pf/libhdll_b200.so > $O/ab_pf.log 2>&1; echo "ab rc=$?"; cat $O/ab_pf.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout=600 -p no:cacheprovider -k "golden or c2 or c3" > $O/gpu_tests_f.log 2>&1; echo "gpu tests rc=$?"; tail -1 $O/gpu_tests_f.log
HDLL_B200_BAND_TIMING=1 timeout 600 python bench.py --config 3 --steps 3 --sigma 1 --tiled --no-cpu > $O/bench_c3_tiled_f.log 2> $O/bench_c3_tiled_f.err; echo "c3 tiled rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"phase_ms_rank0": {[^}]*}' $O/bench_c3_tiled_f.log; tail -12 $O/bench_c3_tiled_f.err
