#!/bin/bash
O=gpurun_out/r2
mkdir -p $O
timeout 300 python tools/pcie.py > $O/pcie.log 2>&1; cat $O/pcie.log
timeout 600 python tools/pipe_timeline.py 10 64 > $O/timeline.json 2> $O/timeline.err; echo rc=$?; head -c 300 $O/timeline.json
