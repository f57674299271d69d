#!/bin/bash
# Default bench line + ncu of the sort kernel.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-q}
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:ng_tile_sort -s 1 -c 1 \
    -o $OUT/prof_sort_$TAG -f python bench.py --grid 256 --rays 64 --precision fp32 --steps 1 --warmup 1 \
    --no-e2e --no-fp32-extra --no-cpu --no-parity > $OUT/ncu_sort_$TAG.log 2>&1
