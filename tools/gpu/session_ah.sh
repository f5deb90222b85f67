#!/bin/bash
# GPU session AH: ncu --set full with source of k_seg_dot on config 3
O=gpurun_out/r2
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_seg_dot" -s 1 -c 1 -o $O/dot_c3_ah python tools/steptimes.py 1 3 2 > $O/ncu_ah.log 2>&1; echo "ncu rc=$?"; tail -1 $O/ncu_ah.log
