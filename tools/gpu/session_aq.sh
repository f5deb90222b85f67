#!/bin/bash
# GPU session AQ: per-kernel instruction / DRAM counts of one c1 step (16 images, host-thread parity model)
O=gpurun_out/r2
mkdir -p $O
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_uniform.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
export HDLL_BLAS_THREADS=16
python tools/steptimes.py 16 1 2 > $O/pl_aq.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file $O/inst_aq.csv python tools/steptimes.py 16 1 2 > $O/ncu_inst_aq.log 2>&1
echo "ncu rc=$?"
