"""Diagnostic: total steps of multigrid solves, fp64/fp32, lean vs register tracers."""
import os, subprocess, sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
code = r'''
import sys, json
sys.path[:0] = ["ROOT", "ROOT/oracle", "ROOT/tests"]
import refshim
from paper_1810_00188_b200 import capi
out = {}
for name, n, v in [("nb-3dimens", 12, dict(n_levels=3, steps_per_level=3)),
                   ("nb-3dimens", 12, dict(n_levels=1)),
                   ("epsw-low", 10, dict(n_levels=2, steps_per_level=4))]:
    g, t, b, m, _ = refshim.ref_case(name, n)
    for prec in (capi.FP64, capi.FP32):
        r = capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=32, seed=77, precision=prec, **v))
        out[f"{name}-{v.get('n_levels')}-{prec}"] = [int(x) for x in r[2]]
    rr = refshim.solve(g, t, b, m, capi.config_struct(rays_per_cell=32, seed=77, **v))
    out[f"{name}-{v.get('n_levels')}-ref"] = [int(x) for x in rr[2]]
print(json.dumps(out))
'''.replace("ROOT", str(ROOT))
for lean in ("1", "0"):
    env = dict(os.environ, ERMC_LEAN=lean)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("lean", lean, r.stdout.strip(), r.stderr[-500:])
