#!/bin/bash
# GPU session: parity subset on the shipped library, A/B of experiment libraries on c1, ncu of the shipped plane coder
# tools/gpu/session_r.sh TAG LIB...
O=gpurun_out/r2
mkdir -p $O
T=$1; shift
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout=600 -p no:cacheprovider -k "plane or golden or wide or config1 or config2" > $O/gpu_tests_$T.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests_$T.log
timeout 1200 python tools/ab.py 64 1 3 6 "$@" > $O/ab_$T.log 2>&1; echo "ab rc=$?"; cat $O/ab_$T.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_entropy_plane" -s 1 -c 1 -o $O/plane64_$T python tools/steptimes.py 64 1 2 > $O/ncu_plane64_$T.log 2>&1
echo "ncu rc=$?"
