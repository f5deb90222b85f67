#!/bin/bash
# GPU session S3B: XU-lean tone map / YCC (exact bit-built RGBE floats, magic-number roundings): all GPU tests, A/B vs the previous build
O=gpurun_out/r2/s3b
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 $O/gpu_tests.log
timeout 1500 python tools/ab.py 64 1 3 6 exp/base0/libhdll_b200.so paper_2309_11072_b200/libhdll_b200.so exp/blmagic/libhdll_b200.so > $O/ab.log 2>&1; echo "ab rc=$?"; cat $O/ab.log
