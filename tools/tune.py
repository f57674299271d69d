"""Scheduling-knob sweep (development aid): runs tools/probe-style timings
for each ERMC_* environment setting in a fresh process."""
import itertools, json, os, subprocess, sys
GRID = int(os.environ.get("TUNE_GRID", "256")); RAYS = int(os.environ.get("TUNE_RAYS", "16"))
code = f"""
import sys, time; sys.path.insert(0, '.')
import torch
from paper_1810_00188_b200 import capi, workloads as W
grid, t, b, m, _ = W.channel_case({GRID}, 'nongrey16')
N = {GRID}**3
tt = torch.from_numpy(t).cuda(); q = torch.empty(N, dtype=torch.float64, device='cuda'); sd = torch.empty_like(q)
st = torch.cuda.current_stream().cuda_stream
out = {{}}
for prec in PRECS:
    s = capi.Session(grid, b, m, capi.config_struct(rays_per_cell={RAYS}, seed=2024, precision=prec))
    s.set_field(tt.data_ptr(), True, st)
    best = 1e30
    for r in range(3):
        steps = s.solve(0, N, q.data_ptr(), sd.data_ptr(), st); ms, nl = s.timings(); best = min(best, ms[2])
    out[prec] = (int(steps.sum()) / (best * 1e-3), best)
    s.close()
print(out)
"""
variants = [v.split(",") for v in sys.argv[1:]] or [[""]]
for v in variants:
    env = dict(os.environ)
    precs = []
    for kv in v:
        if not kv: continue
        k, val = kv.split("=")
        if k == "PREC": precs.append(int(val)); continue
        env[k] = val
    precs = precs or [0, 1]
    r = subprocess.run([sys.executable, "-c", code.replace("PRECS", repr(precs))], env=env, capture_output=True, text=True)
    print(v, r.stdout.strip() or r.stderr[-2000:], flush=True)
