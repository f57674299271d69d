"""Quick throughput probe of the trace kernel (development aid)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1810_00188_b200 import capi, workloads as W

def run(n, rays, prec, model="nongrey16", reps=2):
    grid, t, b, m, _ = W.channel_case(n, model)
    cfg = capi.config_struct(rays_per_cell=rays, seed=2024, precision=prec)
    s = capi.Session(grid, b, m, cfg)
    tt = torch.from_numpy(t).cuda()
    N = n ** 3
    q = torch.empty(N, dtype=torch.float64, device='cuda'); sd = torch.empty_like(q)
    st = torch.cuda.current_stream().cuda_stream
    s.set_field(tt.data_ptr(), True, st)
    for r in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        steps = s.solve(0, N, q.data_ptr(), sd.data_ptr(), st)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        ms, nl = s.timings()
        tot = int(steps.sum())
        print(f"n={n} R={rays} prec={prec} {model}: steps={tot} ({tot/N/rays:.1f}/ray) wall={dt:.3f}s "
              f"trace={ms[2]:.1f}ms reduce={ms[3]:.2f}ms stats={ms[0]:.2f}ms -> {tot/(ms[2]*1e-3):.3e} steps/s (trace), {tot/dt:.3e} (wall)", flush=True)
    s.close()

for prec in (0, 1):
    run(64, 16, prec)
    run(128, 16, prec)
run(256, 16, 1); run(256, 16, 0)
