#!/bin/bash
# GPU session AB: ncu --set full of the four largest kernels (c1, 16 images), per-launch list of one step
O=gpurun_out/r2
mkdir -p $O
python tools/steptimes.py 16 1 2 > $O/pl_ab.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_base_layer|k_entropy_plane|k_sdr_ycc|k_entropy_dct|k_sort_scatter" -s 5 -c 5 -o $O/top5_ab python tools/steptimes.py 16 1 2 > $O/ncu_top5_ab.log 2>&1; echo "ncu full rc=$?"; tail -2 $O/ncu_top5_ab.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ab.csv python tools/steptimes.py 16 1 2 > $O/ncu_l_ab.log 2>&1; echo "ncu list rc=$?"
