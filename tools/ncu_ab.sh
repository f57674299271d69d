#!/bin/bash
# ncu --set full of the fp32/fp64 trace kernel with and without the sorted dispatch,
# plus a launch list of one sorted solve (sort kernel times).
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-x}; PREC=${PREC:-fp32}
for S in ${SORTS:-0 1}; do
  ERMC_SORT=$S timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:trace_pool -s 1 -c 1 \
    -o $OUT/prof_${PREC}_sort${S}_$TAG -f python bench.py --grid 256 --rays 16 --precision $PREC --steps 1 --warmup 1 \
    --no-e2e --no-fp32-extra --cpu-seconds 1 > $OUT/ncu_full_${PREC}_sort${S}_$TAG.log 2>&1
done
ERMC_SORT=1 timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $OUT/ncu_launches_$TAG.csv python bench.py --precision $PREC --steps 1 --warmup 1 --no-e2e --no-fp32-extra --cpu-seconds 1 > /dev/null 2>&1
