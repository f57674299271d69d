#!/bin/bash
# Exercises bench.py's N > 1 flow on a one-GPU box (test only): 2 ranks share
# the GPU and talk over gloo. Also the reference arm under torchrun.
OUT=gpurun_out; mkdir -p $OUT
ERMC_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 --grid 128 --rays 16 \
 --no-cpu --no-single-worker > $OUT/multirank_b200.json 2> $OUT/multirank_b200.err; echo "rc=$?" >> $OUT/multirank_b200.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 \
 --no-cpu --no-single-worker > $OUT/multirank_ref.json 2> $OUT/multirank_ref.err; echo "rc=$?" >> $OUT/multirank_ref.err
cat $OUT/multirank_b200.json $OUT/multirank_ref.json; tail -n 3 $OUT/multirank_b200.err $OUT/multirank_ref.err
