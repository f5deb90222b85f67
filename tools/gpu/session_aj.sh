#!/bin/bash
# GPU session AJ: parity model at the host's 16 OpenBLAS threads -- bench c1 and c3 against the oracle
O=gpurun_out/r2
mkdir -p $O
timeout 900 python bench.py --no-decode > $O/bench_c1_aj.log 2>&1; echo "c1 rc=$?"
timeout 900 python bench.py --config 3 --no-decode > $O/bench_c3_aj.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --config 2 --no-decode > $O/bench_c2_aj.log 2>&1; echo "c2 rc=$?"
for f in $O/bench_c1_aj.log $O/bench_c3_aj.log $O/bench_c2_aj.log; do python - "$f" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print(sys.argv[1], d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'oracle', d.get('parity_vs_oracle'), 'model', d['config'].get('blas_model'), d.get('stage_ms'))
PY
done
