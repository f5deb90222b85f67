#!/bin/bash
# GPU session X: bench lines of every config with the current build (profiles/r02/bench refresh)
O=gpurun_out/r2/x
mkdir -p $O
timeout 900 python bench.py > $O/c1.json.log 2>&1; echo "c1 rc=$?"
timeout 600 python bench.py --sigma 0 --no-decode > $O/c1_s0.json.log 2>&1; echo "c1 s0 rc=$?"
timeout 600 python bench.py --config 0 --no-decode > $O/c0.json.log 2>&1; echo "c0 rc=$?"
timeout 600 python bench.py --config 2 --no-decode > $O/c2.json.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config 21 --no-decode > $O/c21.json.log 2>&1; echo "c21 rc=$?"
timeout 600 python bench.py --config 3 --no-decode > $O/c3.json.log 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --config 3 --tiled --no-decode > $O/c3_tiled.json.log 2>&1; echo "c3 tiled rc=$?"
timeout 600 python bench.py --config 3 --tiled --sigma 0 --no-decode > $O/c3_tiled_s0.json.log 2>&1; echo "c3 tiled s0 rc=$?"
timeout 900 python bench.py --config 4 --steps 3 --no-decode > $O/c4.json.log 2>&1; echo "c4 rc=$?"
for f in $O/*.log; do python - "$f" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], 'NO LINE'); sys.exit()
d=json.loads(l[-1]); pr=d.get('parity_vs_reference',{}); po=d.get('parity_vs_oracle',{})
print(sys.argv[1].split('/')[-1], d.get('value'), d.get('ms_per_step'), 'e2e', (d.get('e2e') or {}).get('value'), 'ref', pr.get('equal'), '/', pr.get('checked'), 'oracle', po.get('equal'), '/', po.get('checked'), 'clk', (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))
PY
done
