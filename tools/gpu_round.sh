#!/bin/bash
# GPU tests + A/B + BASELINE config coverage (tools/configs.py).
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r}
VARIANTS="${VARIANTS:-ERMC_TRACK_POS=0,ERMC_TRACK_POS=1}" PRECS="${PRECS:-fp64}" bash tools/ab.sh $TAG
if [ "${SKIP_CONFIGS:-0}" != "1" ]; then
  rm -f $OUT/configs_$TAG.jsonl
  timeout 1800 python tools/configs.py --out $OUT/configs_$TAG.jsonl ${CONFIG_ARGS:-} > $OUT/configs_$TAG.log 2>&1; echo "configs rc=$?" >> $OUT/configs_$TAG.log
  tail -3 $OUT/configs_$TAG.log
fi
