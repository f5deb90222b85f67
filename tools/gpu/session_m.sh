#!/bin/bash
# GPU session M: full GPU tests on the 4-blocks-per-lane DCT coder; A/B of the plane coder's wave target
O=gpurun_out/r2
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > $O/gpu_tests_m.log 2>&1; echo "gpu tests rc=$?"; tail -1 $O/gpu_tests_m.log
timeout 900 python tools/ab.py 64 1 3 6 exp/pw16/libhdll_b200.so exp/pw8/libhdll_b200.so exp/pw4/libhdll_b200.so > $O/ab_pw_c1.log 2>&1; echo "ab c1 rc=$?"; cat $O/ab_pw_c1.log
timeout 900 python tools/ab.py 1 3 3 6 exp/pw16/libhdll_b200.so exp/pw8/libhdll_b200.so exp/pw32/libhdll_b200.so > $O/ab_pw_c3.log 2>&1; echo "ab c3 rc=$?"; cat $O/ab_pw_c3.log
