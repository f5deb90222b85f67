#!/bin/bash
# GPU session AF: launch list of one c3 step (7680x4320) and one c2 step
O=gpurun_out/r2
mkdir -p $O
python tools/steptimes.py 1 3 2 > $O/pl_af.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_af.csv python tools/steptimes.py 1 3 2 > $O/ncu_af.log 2>&1; echo "ncu c3 rc=$?"
python tools/launches_summary.py $O/launches_c3_af.csv | head -24
