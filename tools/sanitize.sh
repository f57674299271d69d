#!/bin/bash
# compute-sanitizer memcheck / racecheck over small solves of every tracer.
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/san_case.py <<'PY'
import sys
sys.path[:0] = ["ROOT", "ROOT/oracle", "ROOT/tests"]
import numpy as np, refshim
from paper_1810_00188_b200 import capi, workloads as W
cases = [("nb-parab", 10, {}), ("epsw-low", 9, {}), ("nb-3dimens", 10, dict(n_levels=3, steps_per_level=3)),
         ("box-sin-5", 8, dict(specular_walls=1)), ("grey-parab", 8, dict(volume_sampling=1))]
for name, n, v in cases:
    g, t, b, m, _ = refshim.ref_case(name, n)
    for prec in (capi.FP64, capi.FP32):
        capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=8, seed=3, precision=prec, **v))
        capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=8, seed=3, precision=prec, **v), cell_range=(7, 300))
g, t, b, m = W.channel_case(16, "nongrey16")[:4]
for prec in (capi.FP64, capi.FP32):
    capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=8, seed=3, precision=prec, n_devices=2))
    capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=8, seed=3, precision=prec, n_levels=4,
                                              steps_per_level=2))  # black-wall multigrid tracers
g, t, b, m = W.channel_case(32, "nongrey16")[:4]    # 6 levels: the 64-step multigrid window
capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=2, seed=3, n_levels=6, steps_per_level=2))
g, t, b, m = W.channel_case(16, "nongrey119")[:4]   # guides-only CDF staging
for prec in (capi.FP64, capi.FP32):
    capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=8, seed=3, precision=prec))
for mode in (0, 1):                                  # L2 bandwidth probe
    capi.probe_l2(0, 2 << 20, 1, mode)
import paper_1810_00188_b200 as E                    # error raised inside a trace
gr = capi.make_grid((12, 4, 4), (1.0 / 12, 0.25, 0.25))
ma = capi.model_from_ermc(E.grey_model(50.0, E.make_planck_bands(900.0, 1100.0, 8),
                                       E.make_temp_grid(900.0, 1100.0, 10.0)))
ib = ma.ib_table.reshape(ma.n_bands, -1).copy(); ib[:, 3] = np.inf
ma = capi.ModelArrays(ma.nu_lo, ma.nu_hi, ma.nu_center, ma.g_points, ma.g_weights, ma.temps,
                      ma.k_table, ib)
bw = capi.make_boundary((capi.WALL, capi.PERIODIC, capi.PERIODIC), [(950.0, 1.0)] + [(0.0, 1.0)] * 2,
                        [(950.0, 1.0)] + [(0.0, 1.0)] * 2)
tt = np.full(12 * 16, 950.0); tt[8 * 16:] = 925.0
try:
    capi.solve(gr, tt, bw, ma, capi.config_struct(rays_per_cell=8, seed=3))
except capi.ErmcError as e:
    print("expected error:", str(e)[:60])
print("sanitizer cases done")
PY
sed -i "s#ROOT#$PWD#g" /tmp/san_case.py
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san_case.py > $OUT/sanitize_memcheck.txt 2>&1; echo "memcheck rc=$?" >> $OUT/sanitize_memcheck.txt
ERMC_SORT_BLOCK=0 timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san_case.py > $OUT/sanitize_memcheck_blk.txt 2>&1; echo "memcheck rc=$?" >> $OUT/sanitize_memcheck_blk.txt
timeout 1500 $CS --tool racecheck --error-exitcode 9 python /tmp/san_case.py > $OUT/sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?" >> $OUT/sanitize_racecheck.txt
tail -n 3 $OUT/sanitize_memcheck.txt $OUT/sanitize_memcheck_blk.txt $OUT/sanitize_racecheck.txt
