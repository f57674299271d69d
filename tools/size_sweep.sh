#!/bin/bash
# Throughput vs grid size (256^3 is the bench point; 320^3 and 384^3 exceed
# 2^31 work items at R = 64, so the solve runs in chunks).
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-sz}
for N in ${SIZES:-64 128 192 256 320 384}; do for P in fp64 fp32; do
  F=$OUT/size_${TAG}_${N}_$P.json
  timeout 900 python bench.py --grid $N --precision $P --steps 1 --warmup 1 --no-e2e --no-fp32-extra --no-cpu --no-parity > $F 2>&1
  python -c "
import json
d=json.loads(open('$F').read().splitlines()[-1]); print($N, '$P', '%.4g'%d['value'], round(d['roofline']['frac'],3), round(d['ms_per_step'],1), round(d['steps_per_ray'],1))"
done; done
