#!/usr/bin/env python
"""Per-ray setup cost of the trace kernels (measurement aid, not a test).

Solves the bench field (256^3 non-grey channel, R = 64) with the march
capped at max_steps = 1, 2, 4 steps per ray: the trace kernel time is then
almost all ray generation (init_ray + DDA setup + pool refills). Prints one
JSON line per (precision, levels, max_steps) with the trace time and the
implied ns per ray; compare with the uncapped solve of the same config.

    python tools/init_cost.py [--grid 256] [--rays 64]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1810_00188_b200 import capi, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--rays", type=int, default=64)
    ap.add_argument("--levels", default="1,7")
    ap.add_argument("--caps", default="1,2,4,100000")
    ap.add_argument("--precisions", default="fp64")
    a = ap.parse_args()
    g, t, b, m, _ = W.channel_case(a.grid, "nongrey16")
    n = g.nx * g.ny * g.nz
    dev = torch.device("cuda", 0)
    td = torch.from_numpy(t).to(dev)
    q = torch.empty(n, dtype=torch.float64, device=dev)
    sd = torch.empty_like(q)
    for prec in a.precisions.split(","):
        for lv in [int(x) for x in a.levels.split(",")]:
            for cap in [int(x) for x in a.caps.split(",")]:
                cfg = capi.config_struct(rays_per_cell=a.rays, seed=2024, max_steps=cap,
                                         n_levels=lv,
                                         precision=capi.FP64 if prec == "fp64" else capi.FP32)
                s = capi.Session(g, b, m, cfg)
                s.set_field(td.data_ptr(), True, 0)
                s.solve(0, n, q.data_ptr(), sd.data_ptr(), 0)  # warm (builds levels, words)
                best = None
                for _ in range(3):
                    st = s.solve(0, n, q.data_ptr(), sd.data_ptr(), 0)
                    ms = s.timings()[0]
                    best = ms if best is None or ms[2] < best[2] else best
                s.close()
                rays = n * a.rays
                steps = int(np.sum(st))
                print(json.dumps({"precision": prec, "levels": lv, "max_steps": cap,
                                  "trace_ms": best[2], "sort_ms": best[1],
                                  "steps_per_ray": steps / rays,
                                  "ns_per_ray": best[2] * 1e6 / rays,
                                  "ps_per_step": best[2] * 1e9 / steps}), flush=True)


if __name__ == "__main__":
    main()
