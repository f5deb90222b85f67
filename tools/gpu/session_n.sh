#!/bin/bash
# GPU session N (round 2, re-entry): every GPU test, bench c1, ncu launch list of one c1 step
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi_n.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_n.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gpu_tests_n.log
timeout 900 python bench.py > $O/bench_c1_n.log 2>&1; echo "bench c1 rc=$?"; tail -c 3000 $O/bench_c1_n.log
python tools/steptimes.py 16 1 2 > $O/pl_n.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_n.csv python tools/steptimes.py 16 1 2 > $O/ncu_l_n.log 2>&1
echo "ncu rc=$?"
