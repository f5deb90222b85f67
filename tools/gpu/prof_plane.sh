#!/bin/bash
# ncu --set full (source counters) of one k_entropy_plane launch on c1 x16: tools/gpu/prof_plane.sh TAG [LIB]
O=gpurun_out/r2
mkdir -p $O
T=${1:-x}
[ -n "$2" ] && export HDLL_B200_LIB=$PWD/$2
python tools/steptimes.py 16 1 2 > $O/pl_$T.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_entropy_plane" -s 1 -c 1 -o $O/plane_$T python tools/steptimes.py 16 1 2 > $O/ncu_plane_$T.log 2>&1
echo "ncu rc=$?"
