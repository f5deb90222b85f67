#!/bin/bash
# GPU session S3F: ncu --set full of the latency-bound mid-size kernels (k_sdr_ycc, k_prefilter_cols, k_crc_chunks, k_sort_scatter)
O=gpurun_out/r2/s3f
mkdir -p $O
python tools/steptimes.py 16 1 2 > $O/pl.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sdr_ycc|k_prefilter_cols|k_crc_chunks|k_sort_scatter" -s 4 -c 4 -o $O/mid4 python tools/steptimes.py 16 1 2 > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $O/ncu.log
