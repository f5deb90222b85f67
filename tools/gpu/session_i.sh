#!/bin/bash
# GPU session I (round 2): every config's bench line, the reference arm
O=gpurun_out/r2/i
mkdir -p $O
timeout 900 python bench.py > $O/c1.log 2>&1; echo "c1 rc=$?"
timeout 600 python bench.py --sigma 0 --no-decode > $O/c1_s0.log 2>&1; echo "c1 s0 rc=$?"
timeout 1200 python bench.py --config 4 --steps 3 --no-decode > $O/c4.log 2>&1; echo "c4 rc=$?"
timeout 600 python bench.py --config 0 --no-decode > $O/c0.log 2>&1; echo "c0 rc=$?"
for C in 2 21; do timeout 600 python bench.py --config $C --no-decode > $O/c$C.log 2>&1; echo "c$C rc=$?"; done
timeout 600 python bench.py --config 3 --no-decode > $O/c3.log 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --config 3 --tiled > $O/c3_tiled.log 2>&1; echo "c3 tiled rc=$?"
timeout 600 python bench.py --config 3 --tiled --sigma 0 > $O/c3_tiled_s0.log 2>&1; echo "c3 tiled s0 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 > $O/ref.log 2>&1; echo "ref rc=$?"
for f in $O/*.log; do echo "== $f"; grep -o '"value": [0-9.]*, "unit[^,]*, "n_gpus[^,]*\|"ms_per_step": [0-9.]*\|"e2e": {"value": [0-9.]*\|"parity_vs_reference": {[^}]*}' $f | tr '\n' ' '; echo; done
