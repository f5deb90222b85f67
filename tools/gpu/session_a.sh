#!/bin/bash
# GPU session A (round 2): host facts, FP64/ALU ceilings, every GPU test, the
# c1 and c4 bench lines, and a per-kernel instruction / DRAM count pass.
O=gpurun_out/r2
mkdir -p $O
{ nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv;
  python -c "import json,sys; sys.path.insert(0,'.'); from paper_2309_11072_b200.container import host_blas; print(json.dumps(host_blas()))"; } > $O/host.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/peaks tools/peaks_fp64_alu.cu && /tmp/peaks > $O/peaks_fp64_alu.json 2> $O/peaks.err
echo "peaks rc=$?"
timeout 1800 python -m pytest tests -m gpu -q --durations=30 --timeout=600 -p no:cacheprovider > $O/gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -5 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c1.log 2>&1; echo "bench c1 rc=$?"; tail -c 600 $O/bench_c1.log
timeout 1200 python bench.py --config 4 --steps 3 > $O/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -c 300 $O/bench_c4.log
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_uniform.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/steptimes.py 16 1 2 > $O/pl.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file $O/inst.csv python tools/steptimes.py 16 1 2 > $O/ncu_inst.log 2>&1
echo "ncu rc=$?"
