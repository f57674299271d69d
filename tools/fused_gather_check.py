#!/usr/bin/env python
"""Multi-rank check of the fused reduce + all-gather (session_solve_scatter).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/fused_gather_check.py [--grid 32] [--rays 16]

Every rank solves its x-slab; the reduction kernel stores each cell's Q_r /
sigma into every rank's full-field buffer (its own and the peers', mapped with
CUDA IPC). After a barrier each rank's buffer must equal a one-GPU solve of
the whole field byte for byte. Ranks may share a GPU (device = local rank mod
visible devices), so the check also runs on a one-GPU box; the handles and the
barrier go over gloo.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1810_00188_b200 import capi, parallel, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=32)
    ap.add_argument("--rays", type=int, default=16)
    ap.add_argument("--precision", default="fp64")
    a = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    g, t, b, m = W.channel_case(a.grid, "nongrey16")[:4]
    n = g.nx * g.ny * g.nz
    prec = capi.FP64 if a.precision == "fp64" else capi.FP32
    cfg = capi.config_struct(rays_per_cell=a.rays, seed=99, precision=prec, device=dev)
    slab = parallel.x_slab(g.nx, g.ny, g.nz, world, rank)

    q_full = capi.device_alloc(dev, n * 8)
    sd_full = capi.device_alloc(dev, n * 8)
    handles = [None] * world
    dist.all_gather_object(handles, (capi.ipc_export(q_full), capi.ipc_export(sd_full)))
    outs_q, outs_sd = [], []
    for r in range(world):
        if r == rank:
            outs_q.append(q_full)
            outs_sd.append(sd_full)
        else:
            outs_q.append(capi.ipc_open(handles[r][0]))
            outs_sd.append(capi.ipc_open(handles[r][1]))

    td = torch.from_numpy(t).cuda(dev)
    s = capi.Session(g, b, m, cfg)
    s.set_field(td.data_ptr(), True, 0)
    steps = s.solve_scatter(slab.lo, slab.hi, outs_q, outs_sd, 0)
    torch.cuda.synchronize(dev)
    dist.barrier()

    q = torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}")
    sd = torch.empty_like(q)
    import ctypes as C  # noqa: PLC0415
    cudart = C.CDLL("libcudart.so")
    cudart.cudaMemcpy(C.c_void_p(q.data_ptr()), C.c_void_p(q_full), C.c_size_t(n * 8), 3)
    cudart.cudaMemcpy(C.c_void_p(sd.data_ptr()), C.c_void_p(sd_full), C.c_size_t(n * 8), 3)
    qh, sdh = q.cpu().numpy(), sd.cpu().numpy()
    ref_q, ref_sd, _, ref_total, _ = capi.solve(g, t, b, m, cfg)
    tot = torch.tensor([int(steps.sum())], dtype=torch.int64)
    dist.all_reduce(tot)
    ok = bool(np.array_equal(qh, ref_q) and np.array_equal(sdh, ref_sd)
              and int(tot.item()) == ref_total)
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    if rank == 0:
        print(json.dumps({"world": world, "grid": a.grid, "rays": a.rays,
                          "precision": a.precision, "byte_identical_on_every_rank": oks,
                          "total_steps": int(tot.item()), "reference_total": ref_total}))
    s.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if all(oks) else 1)


if __name__ == "__main__":
    main()
