#!/bin/bash
# ncu --set full of one k_entropy_plane launch on c1 x64 for two libraries: tools/gpu/prof_plane64.sh TAG LIB_A LIB_B
O=gpurun_out/r2
mkdir -p $O
T=$1
for L in $2 $3; do
  n=$(basename $(dirname $L))
  HDLL_B200_LIB=$PWD/$L timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_entropy_plane" -s 1 -c 1 -o $O/plane64_${T}_$n python tools/steptimes.py 64 1 2 > $O/ncu_plane64_${T}_$n.log 2>&1
  echo "ncu $n rc=$?"
done
