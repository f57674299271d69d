#!/bin/bash
# A/B of the narrow-band sorted dispatch (ERMC_SORT, ERMC_SORT_TILE) on the bench workload.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-ab}
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
fi
for V in ${VARIANTS:-"0 65536" "1 16384" "1 65536" "1 262144"}; do set -- $V; for P in ${PRECS:-fp64 fp32}; do
  ERMC_SORT=$1 ERMC_SORT_TILE=$2 timeout 600 python bench.py --precision $P --steps 2 --warmup 3 --no-e2e --no-fp32-extra --cpu-seconds 1 > $OUT/bench_${TAG}_s$1_t$2_$P.json 2>&1
  echo "sort=$1 tile=$2 $P $(python -c "
import json,sys
d=json.loads(open('$OUT/bench_${TAG}_s$1_t$2_$P.json').read().splitlines()[-1]); print('%.4g'%d['value'], d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], d['ms_per_step'])")"
done; done
