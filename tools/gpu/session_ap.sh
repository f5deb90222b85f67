#!/bin/bash
# GPU session AP: ddot launch shape by batch size -- parity subset, A/B c1 (1 and 16 threads), c3 (16), bench c4 (host threads)
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tiled.py -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_ap.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests_ap.log
H=exp/head/libhdll_b200.so; C=exp/cur/libhdll_b200.so
timeout 1200 python tools/ab.py 64 1 3 5 $H,HDLL_BLAS_THREADS=16 $C,HDLL_BLAS_THREADS=16 $H $C > $O/ab_ap.log 2>&1; echo "c1 rc=$?"; cat $O/ab_ap.log
timeout 1200 python tools/ab.py 1 3 3 5 $H,HDLL_BLAS_THREADS=16 $C,HDLL_BLAS_THREADS=16 > $O/ab_ap3.log 2>&1; echo "c3 rc=$?"; cat $O/ab_ap3.log
timeout 900 python bench.py --config 4 --steps 3 --no-decode --no-cpu > $O/bench_c4_ap.log 2>&1; echo "c4 rc=$?"; python - <<'PY'
import json
l=[x for x in open('gpurun_out/r2/bench_c4_ap.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['config'].get('blas_model'), d.get('stage_ms'))
PY
