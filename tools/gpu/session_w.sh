#!/bin/bash
# GPU session W: ncu --set full of the serial decoder (decode_sdr of one config-1 image)
O=gpurun_out/r2
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_coders -c 1 -o $O/dec_${TAG:-sdr}_w python tools/decode_one.py $ARGS > $O/ncu_dec_w.log 2>&1; echo "ncu rc=$?"; tail -3 $O/ncu_dec_w.log
