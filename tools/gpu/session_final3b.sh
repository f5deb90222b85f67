#!/bin/bash
# GPU session FINAL3b: the ncu launch list of the bench command itself (python bench.py --steps 2 --warmup 3, config 1, 64 images),
# taken after the same command has exited 0 without ncu; per-kernel shares by tools/launches_summary.py
O=gpurun_out/r2/final3
mkdir -p $O
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-decode > $O/bench_for_launches.json.log 2>&1; rc=$?; echo "bench rc=$rc"
[ $rc -eq 0 ] && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-decode > $O/ncu_bench.log 2>&1; echo "ncu bench list rc=$?"
python tools/launches_summary.py $O/launches_bench.csv > $O/launches_bench.txt 2>&1; head -30 $O/launches_bench.txt
