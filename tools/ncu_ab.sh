#!/bin/bash
# ncu --set full of one trace launch per variant (env VARIANTS: comma-separated
# "PREC SORT BRICK" triples), 256^3 channel, R = 16.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-x}
IFS=',' read -ra VS <<< "${VARIANTS:-fp64 1 0,fp64 1 1}"
for V in "${VS[@]}"; do set -- $V
  ERMC_SORT=$2 ERMC_BRICK=$3 timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:trace_pool -s 1 -c 1 \
    -o $OUT/prof_$1_s$2_b$3_$TAG -f python bench.py --grid 256 --rays 16 --precision $1 --steps 1 --warmup 1 \
    --no-e2e --no-fp32-extra --cpu-seconds 1 > $OUT/ncu_full_$1_s$2_b$3_$TAG.log 2>&1
done
if [ -n "${HOSTPROF:-}" ]; then
  ERMC_HOST_PROFILE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-fp32-extra --cpu-seconds 1 > $OUT/bench_hostprof_$TAG.json 2> $OUT/bench_hostprof_$TAG.err
fi
