#!/bin/bash
# A/B of tuning knobs on the bench workload (results never depend on them).
# VARIANTS: comma-separated lists of env assignments, e.g.
#   VARIANTS="ERMC_CACHE_HINT=0,ERMC_CACHE_HINT=1 ERMC_SORT=0" bash tools/ab.sh tag
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-ab}
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
  tail -2 $OUT/pytest_gpu_$TAG.log
fi
IFS=',' read -ra VS <<< "${VARIANTS:-ERMC_SORT=1}"
i=0
for V in "${VS[@]}"; do for P in ${PRECS:-fp64 fp32}; do
  F=$OUT/bench_${TAG}_v${i}_$P.json
  env $V timeout 600 python bench.py --precision $P --steps 2 --warmup 3 --no-e2e --no-fp32-extra --no-cpu --no-parity ${BENCH_ARGS:-} > $F 2>&1
  echo "[$V] $P $(python -c "
import json,sys
d=json.loads(open('$F').read().splitlines()[-1]); print('%.4g'%d['value'], '%.4f'%d['roofline']['frac'], '%.1f'%d['roofline']['kernel_ms_per_step'], '%.1f'%d['ms_per_step'])")"
done; i=$((i+1)); done
