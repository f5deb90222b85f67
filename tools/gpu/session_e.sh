#!/bin/bash
# GPU session E (round 2): sigma-0 fit (per-pixel shared atomics), tiled phase split
O=gpurun_out/r2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_tiled.py tests/test_gpu_parity.py -q -x --timeout=600 -p no:cacheprovider -k "s0 or tiled or golden" > $O/gpu_tests_e.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gpu_tests_e.log
timeout 600 python bench.py --sigma 0 --no-decode --no-cpu > $O/bench_c1_s0_e.log 2>&1; echo "c1 s0 rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}\|"parity_vs_reference": {[^}]*}' $O/bench_c1_s0_e.log
timeout 600 python bench.py --config 3 --steps 5 --sigma 0 --no-decode --no-cpu > $O/bench_c3_plain_e_s0.log 2>&1; echo "c3 plain s0 rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' $O/bench_c3_plain_e_s0.log
timeout 600 python bench.py --config 3 --steps 5 --sigma 1 --tiled --no-cpu > $O/bench_c3_tiled_e_s1.log 2>&1; echo "c3 tiled s1 rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"phase_ms_rank0": {[^}]*}' $O/bench_c3_tiled_e_s1.log
