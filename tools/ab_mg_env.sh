#!/bin/bash
# Multigrid A/B of env knobs (timing only, no CPU parity samples):
#   VARIANTS="ERMC_INNER_STEPS=32,ERMC_INNER_STEPS=16" LEVELS=4,7 bash tools/ab_mg_env.sh tag
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-mge}
IFS=',' read -ra VS <<< "${VARIANTS:-ERMC_SORT=1}"
for rep in 1 2; do i=0; for V in "${VS[@]}"; do
  F=$OUT/mge_${TAG}_v${i}_$rep.jsonl; rm -f $F
  env $V timeout 900 python tools/configs.py --only mg --mg-levels ${LEVELS:-4,7} \
      --mg-precisions ${PRECS:-fp64,fp32} --no-cpu-check --out $F > /dev/null 2>&1
  python -c "
import json
for l in open('$F'):
    d=json.loads(l)
    print('[$V]', $rep, d['precision'], d['n_levels'], round(d['solve_ms'],1), '%.3g'%d['trace_steps_per_s'])
"
  i=$((i+1)); done; done
