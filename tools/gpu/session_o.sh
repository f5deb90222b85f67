#!/bin/bash
# GPU session O: ncu --set full (source counters) of the plane coder, base layer and sort scatter on c1 x16
O=gpurun_out/r2
mkdir -p $O
python tools/steptimes.py 16 1 2 > $O/pl_o.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_entropy_plane|k_base_layer|k_sort_scatter|k_sdr_ycc" -s 4 -c 4 -o $O/full_o python tools/steptimes.py 16 1 2 > $O/ncu_o.log 2>&1
echo "ncu rc=$?"; tail -3 $O/ncu_o.log
