#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture.
# Usage (from repo root, under gpurun): bash tools/gpu_session.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
fi
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
fi
if [ "${SKIP_NCU:-0}" != "1" ]; then
  NCU=/usr/local/cuda/bin/ncu
  timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $OUT/ncu_launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > $OUT/ncu_launches_bench_$TAG.json 2>&1
  for P in fp64 fp32; do
    timeout 900 $NCU --set full --clock-control none --import-source on -k regex:trace_pool -s 1 -c 1 \
      -o $OUT/prof_${P}_$TAG -f python bench.py --grid 256 --rays 16 --precision $P --steps 1 --warmup 1 \
      --no-e2e --no-fp32-extra --no-cpu --no-parity > $OUT/ncu_full_${P}_$TAG.log 2>&1
  done
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:ng_tile_sort -s 1 -c 1 \
    -o $OUT/prof_sort_$TAG -f python bench.py --grid 256 --rays 64 --precision fp32 --steps 1 --warmup 1 \
    --no-e2e --no-fp32-extra --no-cpu --no-parity > $OUT/ncu_sort_$TAG.log 2>&1
fi
if [ "${SKIP_CONFIGS:-1}" != "1" ]; then
  rm -f $OUT/configs_$TAG.jsonl
  timeout 1800 python tools/configs.py --out $OUT/configs_$TAG.jsonl > $OUT/configs_$TAG.log 2>&1; echo "configs rc=$?" >> $OUT/configs_$TAG.log
fi
ls -la $OUT
