#!/bin/bash
# GPU session P2: e2e pipeline timeline (c1, 64-image chunks, 10 repeats) and the PCIe copy rates
O=gpurun_out/r2
mkdir -p $O
timeout 600 python tools/pipe_timeline.py 10 64 > $O/pipe_tl.json 2>&1; echo "tl rc=$?"
timeout 300 python tools/pcie.py > $O/pcie.log 2>&1; echo "pcie rc=$?"; tail -5 $O/pcie.log
