#!/bin/bash
# GPU session AE: ncu --set full with source of k_seg_nodes and k_prefilter_cols (c1, 16 images)
O=gpurun_out/r2
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_seg_nodes|k_prefilter_cols|k_tm_nodes" -s 3 -c 3 -o $O/nodes_ae python tools/steptimes.py 16 1 2 > $O/ncu_ae.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu_ae.log
