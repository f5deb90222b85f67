#!/bin/bash
# per-kernel device time of one encode step (cold-cache, serialised by ncu): tools/launches.sh NIMG [CONFIG]
N=${1:-16}
C=${2:-1}
python tools/steptimes.py $N $C 2 > gpurun_out/pl.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/steptimes.py $N $C 2 > gpurun_out/ncu_l.log 2>&1
