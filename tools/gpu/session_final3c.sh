#!/bin/bash
# GPU session FINAL3c: the bench's N > 1 plumbing (NCCL process group, barriers, max / sum all-reduces, digest gather)
# exercised on the one GPU at world size 1 (HDLL_BENCH_FORCE_DIST=1), and the same through torchrun --nproc-per-node 1
O=gpurun_out/r2/final3
mkdir -p $O
HDLL_BENCH_FORCE_DIST=1 NCCL_DEBUG=WARN timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-decode > $O/c1_forcedist.json.log 2>&1; echo "force-dist rc=$?"
HDLL_BENCH_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-decode > $O/c1_torchrun1.json.log 2>&1; echo "torchrun rc=$?"
HDLL_BENCH_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --gpus 1 --config 3 --tiled --steps 3 --warmup 3 --no-cpu --no-decode > $O/c3_tiled_torchrun1.json.log 2>&1; echo "torchrun tiled rc=$?"
for f in c1_forcedist c1_torchrun1 c3_tiled_torchrun1; do grep '^{' $O/$f.json.log | tail -1 | cut -c1-330; tail -2 $O/$f.json.log | grep -v '^{' | cut -c1-300; done
