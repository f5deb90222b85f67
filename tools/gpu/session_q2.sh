#!/bin/bash
# GPU session Q2: pipeline tests, bench c1 and c4 with mapped lengths and the c/4..3c/4 ramp
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_plugin.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_q2.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_q2.log
timeout 900 python bench.py --no-decode > $O/bench_c1_q2.log 2>&1; echo "c1 rc=$?"
timeout 900 python bench.py --config 4 --steps 3 --no-decode > $O/bench_c4_q2.log 2>&1; echo "c4 rc=$?"
for f in $O/bench_c1_q2.log $O/bench_c4_q2.log; do python - "$f" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print(sys.argv[1], d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e'].get('streams_equal_device_run'), (d.get('parity_vs_reference') or {}).get('equal'))
PY
done
