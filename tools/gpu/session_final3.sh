#!/bin/bash
# GPU session FINAL3 (round-end state after the k_sdr_ycc straight-line tone-map block): every GPU test, smoke, bench lines of every config, the reference arm,
# launch list of one c1 step and ncu --set full of the five largest kernels
O=gpurun_out/r2/final3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/c1.json.log 2>&1; echo "c1 rc=$?"
timeout 600 python bench.py --impl reference > $O/ref.json.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --sigma 0 --no-decode > $O/c1_s0.json.log 2>&1; echo "c1 s0 rc=$?"
timeout 600 python bench.py --config 0 --no-decode > $O/c0.json.log 2>&1; echo "c0 rc=$?"
timeout 600 python bench.py --config 2 --no-decode > $O/c2.json.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config 21 --no-decode > $O/c21.json.log 2>&1; echo "c21 rc=$?"
timeout 600 python bench.py --config 3 --no-decode > $O/c3.json.log 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --config 3 --tiled --no-decode > $O/c3_tiled.json.log 2>&1; echo "c3 tiled rc=$?"
timeout 600 python bench.py --config 3 --tiled --sigma 0 --no-decode > $O/c3_tiled_s0.json.log 2>&1; echo "c3 tiled s0 rc=$?"
timeout 900 python bench.py --config 4 --steps 3 --no-decode > $O/c4.json.log 2>&1; echo "c4 rc=$?"
for f in $O/*.json.log; do python - "$f" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], 'NO LINE'); sys.exit()
d=json.loads(l[-1]); pr=d.get('parity_vs_reference') or {}; po=d.get('parity_vs_oracle') or {}
print(sys.argv[1].split('/')[-1], d.get('value'), d.get('ms_per_step'), 'e2e', (d.get('e2e') or {}).get('value'), 'ref', pr.get('equal'), '/', pr.get('checked'), 'oracle', po.get('equal'), '/', po.get('checked'), 'clk', (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))
PY
done
python tools/steptimes.py 16 1 2 > $O/pl.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1x16.csv python tools/steptimes.py 16 1 2 > $O/ncu_l.log 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_base_layer|k_entropy_plane|k_sdr_ycc|k_entropy_dct|k_sort_scatter" -s 5 -c 5 -o $O/top5 python tools/steptimes.py 16 1 2 > $O/ncu_top5.log 2>&1; echo "ncu full rc=$?"
