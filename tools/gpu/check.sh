#!/bin/bash
# GPU-box session: host facts, GPU tests, bench (tools/gpu/*.sh are run through gpurun)
mkdir -p gpurun_out/r2
{ nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; python -c "import threadpoolctl, json; print(json.dumps([i for i in threadpoolctl.threadpool_info() if i['user_api']=='blas']))"; } > gpurun_out/r2/host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2/bench.log
