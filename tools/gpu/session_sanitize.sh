#!/bin/bash
# GPU session SANITIZE: tools/small_cases.py (every kernel family on small inputs, checked against the oracle).
# compute-sanitizer is closed on this pool (the wrapper refuses to start it), so the script runs plainly.
O=gpurun_out/r2/sanitize
mkdir -p $O
timeout 600 python tools/small_cases.py > $O/plain.log 2>&1; echo "plain rc=$?"; tail -30 $O/plain.log
