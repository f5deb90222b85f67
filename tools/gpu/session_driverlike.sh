#!/bin/bash
# GPU session DRIVERLIKE: the driver's round-end commands as round 1 ran them (reference arm first, then this arm), wall-clocked
O=gpurun_out/r2/final3
mkdir -p $O
timeout 1200 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/driver_ref.json.log 2>&1; echo "ref rc=$? at ${SECONDS}s"
timeout 1200 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/driver_c1.json.log 2>&1; echo "c1 rc=$? at ${SECONDS}s"
python - <<'PY'
import json
O='gpurun_out/r2/final3/'
r=json.loads([l for l in open(O+'driver_ref.json.log') if l.startswith('{')][-1])
c=json.loads([l for l in open(O+'driver_c1.json.log') if l.startswith('{')][-1])
print('reference', r['value'], r['unit'], 'ms/step', r['ms_per_step'])
print('b200', c['value'], 'e2e', c['e2e']['value'], 'ms/step', c['ms_per_step'], 'clocks', c['clocks'], 'parity', c['parity_vs_reference'], c['parity_vs_oracle'])
print('ratio value', c['value']/r['value'], 'e2e', c['e2e']['value']/r['e2e']['value'])
PY
