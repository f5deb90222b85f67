#!/bin/bash
# GPU session Z2: c4 like-sized batches; CRC (warp over 32-unit groups) A/B on c1 and parity subset
O=gpurun_out/r2
mkdir -p $O
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-decode --no-cpu --batch-order size > $O/c4_size.log 2>&1; echo "c4 size rc=$?"
for f in $O/c4_size.log; do python - "$f" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print(sys.argv[1], d['value'], d['ms_per_step'], (d.get('parity_vs_reference') or {}).get('equal'), d.get('stage_ms'))
PY
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -p no:cacheprovider -k "golden" > $O/gpu_tests_crc2.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_crc2.log
timeout 1200 python tools/ab.py 64 1 3 6 exp/head/libhdll_b200.so exp/cur/libhdll_b200.so > $O/ab_crc2.log 2>&1; echo "ab rc=$?"; cat $O/ab_crc2.log
