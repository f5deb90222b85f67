#!/bin/bash
O=gpurun_out/r2
mkdir -p $O
nvidia-smi -i 0 --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > $O/smi_bg.txt &
P=$!
timeout 300 python tools/tiled_diag.py > $O/tdiag4.log 2>&1; echo rc=$?; grep step $O/tdiag4.log | cut -c1-120
kill $P
timeout 300 python bench.py --config 3 --steps 5 --tiled --no-cpu > $O/bench_c3_tiled_h.log 2>&1; echo rc=$?; grep -o '"ms_per_step": [0-9.]*\|"phase_ms_rank0": {[^}]*}' $O/bench_c3_tiled_h.log
