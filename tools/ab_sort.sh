#!/bin/bash
# A/B of scheduling knobs on the bench workload.
# VARIANTS: comma-separated "SORT TILE BRICK" triples, e.g. "0 65536 1,1 65536 1".
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-ab}
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -2 $OUT/pytest_gpu_$TAG.log
fi
IFS=',' read -ra VS <<< "${VARIANTS:-0 65536 1,1 65536 1}"
for V in "${VS[@]}"; do set -- $V; for P in ${PRECS:-fp64 fp32}; do
  F=$OUT/bench_${TAG}_s$1_t$2_b$3_$P.json
  ERMC_SORT=$1 ERMC_SORT_TILE=$2 ERMC_BRICK=$3 timeout 600 python bench.py --precision $P --steps 2 --warmup 3 --no-e2e --no-fp32-extra --cpu-seconds 1 > $F 2>&1
  echo "sort=$1 tile=$2 brick=$3 $P $(python -c "
import json,sys
d=json.loads(open('$F').read().splitlines()[-1]); print('%.4g'%d['value'], '%.4f'%d['roofline']['frac'], '%.1f'%d['roofline']['kernel_ms_per_step'], '%.1f'%d['ms_per_step'])")"
done; done
