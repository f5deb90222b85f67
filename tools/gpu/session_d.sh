#!/bin/bash
# GPU session D (round 2): sigma-0 fit, tiled phases, ncu --set full of the base / sort / DCT-coder kernels
O=gpurun_out/r2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_tiled.py -q -x --timeout=600 -p no:cacheprovider -k "s0 or tiled" > $O/gpu_tests_d.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gpu_tests_d.log
for S in 0 1; do
  timeout 600 python bench.py --config 3 --steps 5 --sigma $S --no-decode --no-cpu > $O/bench_c3_plain_d_s$S.log 2>&1; echo "c3 plain s$S rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' $O/bench_c3_plain_d_s$S.log
  timeout 600 python bench.py --config 3 --steps 5 --sigma $S --tiled --no-cpu > $O/bench_c3_tiled_d_s$S.log 2>&1; echo "c3 tiled s$S rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"phase_ms_rank0": {[^}]*}\|"parity_vs_reference": {[^}]*}' $O/bench_c3_tiled_d_s$S.log
done
timeout 600 python bench.py --sigma 0 --no-decode --no-cpu > $O/bench_c1_s0.log 2>&1; echo "c1 s0 rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}\|"parity_vs_reference": {[^}]*}' $O/bench_c1_s0.log
python tools/steptimes.py 16 1 2 > $O/pl_d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_base_layer|k_sdr_ycc|k_sort_scatter|k_entropy_dct" -s 4 -c 4 -o $O/stages_full python tools/steptimes.py 16 1 2 > $O/ncu_stages.log 2>&1
echo "ncu rc=$?"
