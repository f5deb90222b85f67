#!/bin/bash
O=gpurun_out/r2
mkdir -p $O
HDLL_B200_BAND_TIMING=1 timeout 600 python bench.py --config 3 --steps 3 --sigma 1 --tiled --no-cpu > $O/bench_c3_tiled_g.log 2> $O/bench_c3_tiled_g.err; echo "c3 tiled rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"phase_ms_rank0": {[^}]*}' $O/bench_c3_tiled_g.log; grep "band_begin\|encode_band" $O/bench_c3_tiled_g.err | tail -14
