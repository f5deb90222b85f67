#!/bin/bash
# GPU session C (round 2): GPU tests, bench c1, c3 plain / tiled at sigma 1 and 0,
# ncu --set full of the base-layer, fit-sort and DCT-coder kernels
O=gpurun_out/r2
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_c.log 2>&1; echo "gpu tests rc=$?"; tail -3 $O/gpu_tests_c.log
timeout 900 python bench.py --no-decode > $O/bench_c1_c.log 2>&1; echo "bench c1 rc=$?"; grep -o '"value": [0-9.]*, "unit[^,]*, "n_gpus[^,]*, "steps[^,]*, "warmup[^,]*, "ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}\|"e2e": {"value": [0-9.]*' $O/bench_c1_c.log
for S in 1 0; do
  timeout 600 python bench.py --config 3 --steps 5 --sigma $S --no-decode --no-cpu > $O/bench_c3_plain_s$S.log 2>&1; echo "c3 plain s$S rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' $O/bench_c3_plain_s$S.log
  timeout 600 python bench.py --config 3 --steps 5 --sigma $S --tiled --no-cpu > $O/bench_c3_tiled_s$S.log 2>&1; echo "c3 tiled s$S rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"parity_vs_reference": {[^}]*}' $O/bench_c3_tiled_s$S.log
done
python tools/steptimes.py 16 1 2 > $O/pl_c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_base_layer|k_sdr_ycc|k_sort_scatter|k_entropy_dct" -s 8 -c 4 -o $O/stages_full python tools/steptimes.py 16 1 2 > $O/ncu_stages.log 2>&1
echo "ncu rc=$?"
