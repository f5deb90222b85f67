#!/bin/bash
# GPU session B (round 2): A/B of the per-chain coder modes, bench c1 (with
# decode timing), c3 plain / tiled on one rank, ncu --set full of k_entropy_plane
O=gpurun_out/r2
mkdir -p $O
timeout 900 python tools/ab.py 64 1 3 6 exp/cur/libhdll_b200.so exp/nocmode/libhdll_b200.so > $O/ab_cmode.log 2>&1; echo "ab rc=$?"; cat $O/ab_cmode.log
timeout 900 python bench.py > $O/bench_c1_b.log 2>&1; echo "bench c1 rc=$?"; tail -c 1500 $O/bench_c1_b.log
timeout 600 python bench.py --config 3 --steps 5 --no-decode > $O/bench_c3_plain.log 2>&1; echo "c3 plain rc=$?"; grep -o '"value": [0-9.]*, "unit[^,]*, "n_gpus[^,]*, "steps[^,]*, "warmup[^,]*, "ms_per_step": [0-9.]*' $O/bench_c3_plain.log
timeout 600 python bench.py --config 3 --steps 5 --tiled > $O/bench_c3_tiled.log 2>&1; echo "c3 tiled rc=$?"; tail -c 1200 $O/bench_c3_tiled.log
timeout 600 python bench.py --config 3 --steps 5 --tiled --sigma 0 > $O/bench_c3_tiled_s0.log 2>&1; echo "c3 tiled s0 rc=$?"; grep -o '"ms_per_step": [0-9.]*' $O/bench_c3_tiled_s0.log; grep -o '"parity_vs_reference": {[^}]*}' $O/bench_c3_tiled_s0.log
timeout 600 python bench.py --config 3 --steps 5 --sigma 0 --no-decode > $O/bench_c3_plain_s0.log 2>&1; echo "c3 plain s0 rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"fit": [0-9.]*' $O/bench_c3_plain_s0.log
python tools/steptimes.py 16 1 2 > $O/pl_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_entropy_plane -s 1 -c 1 -o $O/plane_full python tools/steptimes.py 16 1 2 > $O/ncu_plane.log 2>&1
echo "ncu rc=$?"
