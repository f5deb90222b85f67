#!/bin/bash
# GPU session Z: c4 batch composition (stream order vs like-sized batches); CRC A/B on c1 and parity subset
O=gpurun_out/r2
mkdir -p $O
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-decode --no-cpu > $O/c4_stream.log 2>&1; echo "c4 stream rc=$?"
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-decode --no-cpu --batch-order size > $O/c4_size.log 2>&1; echo "c4 size rc=$?"
for f in $O/c4_stream.log $O/c4_size.log; do python - "$f" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print(sys.argv[1], d['value'], d['ms_per_step'], (d.get('parity_vs_reference') or {}).get('equal'), d.get('stage_ms'))
PY
done
TAG=crc bash tools/gpu/session_y.sh
