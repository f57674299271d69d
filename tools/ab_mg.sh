#!/bin/bash
# Multigrid A/B of library builds: LIBS="a.so,b.so" bash tools/ab_mg.sh tag
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-mg}
IFS=',' read -ra LS <<< "${LIBS}"
for rep in 1 2; do for L in "${LS[@]}"; do
  F=$OUT/mg_${TAG}_$(basename $L .so)_$rep.jsonl; rm -f $F
  ERMC_B200_LIB=$L timeout 900 python tools/configs.py --only mg --out $F > /dev/null 2>&1
  python -c "
import json
for l in open('$F'):
    d=json.loads(l)
    if d['n_levels']>1: print('$L', $rep, d['precision'], d['n_levels'], round(d['solve_ms'],1), '%.3g'%d['trace_steps_per_s'], d.get('cpu_parity',{}).get('frac_within_tol'))
"
done; done
