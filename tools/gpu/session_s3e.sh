#!/bin/bash
# GPU session S3E: CRC chunks with 64 bytes per lane in flight (plain / evict-first loads)
O=gpurun_out/r2/s3e
mkdir -p $O
timeout 2000 python tools/ab.py 64 1 3 6 paper_2309_11072_b200/libhdll_b200.so exp/crcpf/libhdll_b200.so exp/crcpfcs/libhdll_b200.so > $O/ab.log 2>&1; echo "ab rc=$?"; cat $O/ab.log
