#!/bin/bash
# A/B of two builds of libermc_b200.so in one GPU session (same box, same
# clocks): LIBS="path1,path2" PRECS="fp64" bash tools/ab_lib.sh tag
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-abl}
IFS=',' read -ra LS <<< "${LIBS}"
for rep in 1 2; do
for L in "${LS[@]}"; do for P in ${PRECS:-fp64}; do
  F=$OUT/bench_${TAG}_$(basename $L .so)_${P}_$rep.json
  ERMC_B200_LIB=$L timeout 600 python bench.py --precision $P --steps 2 --warmup 3 --no-e2e --no-fp32-extra --no-cpu --no-parity ${BENCH_ARGS:-} > $F 2>&1
  echo "[$L rep $rep] $P $(python -c "
import json
d=json.loads(open('$F').read().splitlines()[-1]); print('%.4g'%d['value'], '%.4f'%d['roofline']['frac'], '%.1f'%d['roofline']['kernel_ms_per_step'])")"
done; done; done
