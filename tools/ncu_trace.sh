#!/bin/bash
# ncu --set full of one trace launch per precision (256^3, R=4 keeps replays short).
TAG=${1:-x}; OUT=gpurun_out; mkdir -p $OUT
for P in fp64 fp32; do
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:trace_pool -s 1 -c 1 \
    -o $OUT/prof_${P}_$TAG -f python bench.py --grid 256 --rays 4 --precision $P --steps 1 --warmup 1 \
    --no-e2e --no-fp32-extra --cpu-seconds 1 > $OUT/ncu_full_${P}_$TAG.log 2>&1
done
python - <<'PY' > $OUT/l2_attrs_$TAG.txt 2>&1
import torch
p = torch.cuda.get_device_properties(0)
print(p)
import ctypes
cudart = ctypes.CDLL("libcudart.so")
for name, attr in (("MaxPersistingL2CacheSize", 108), ("L2CacheSize", 38), ("MaxSharedMemoryPerMultiprocessor", 81)):
    v = ctypes.c_int()
    cudart.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(name, v.value)
PY
