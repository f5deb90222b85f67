#!/bin/bash
# GPU session T (round 2, third re-entry): every GPU test, smoke, bench c1, ncu launch list of one c1 step
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi_t.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_t.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gpu_tests_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_t.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_t.log
timeout 900 python bench.py > $O/bench_c1_t.log 2>&1; echo "bench c1 rc=$?"; tail -c 3000 $O/bench_c1_t.log
python tools/steptimes.py 16 1 2 > $O/pl_t.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_t.csv python tools/steptimes.py 16 1 2 > $O/ncu_l_t.log 2>&1
echo "ncu rc=$?"
