#!/usr/bin/env python
"""Every BASELINE.json config on one B200, with its accuracy check.

    python tools/configs.py [--out gpurun_out/configs.jsonl] [--only c1,c4]

One JSON line per run: workload, precision, device time of the solve (CUDA
events around the session call, inputs resident in HBM) and of the trace
kernel, ray-cell steps/s, steps per ray, and the check that applies:
  c1  config 1: 32^3 isothermal grey slab between cold black plates vs the
      closed-form slab solution (oracle/ermc_oracle.c slab_oracle);
  c2  config 2: 128^3 grey channel, tau in {0.1, 0.3, 1, 3, 10};
  c3  config 3: 128^3 non-grey channel, 16 and 119 bands x 16 g;
  c4  config 4: 256^3 non-grey channel (the bench workload), fp64 and fp32;
  c5  config 5: rays-per-cell sweep at 256^3 — max / median sigma and time
      vs R, with log-log slopes (expected -0.5 and ~1);
  full  a whole 128^3 config-3 field against the reference's solve() (every
      cell, every step count);
  mg  multigrid ray coarsening (n_levels 1..7) on the config-4 field.
Channel runs are checked per cell against the reference CPU solver
(oracle/_ref, cell-subset replay — bitwise its solve() for those cells) on
a stratified sample of cells; fp32 runs against the fp64 solve (3 sigma).
Test/measurement infrastructure: imports oracle/ only as the checker.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "oracle"), str(ROOT / "tests")]

import torch  # noqa: E402

import oracle  # noqa: E402
import refshim  # noqa: E402
import paper_1810_00188_b200 as E  # noqa: E402
from helpers import allowed_3sigma, fp64_report, three_sigma_violations  # noqa: E402
from paper_1810_00188_b200 import capi, workloads as W  # noqa: E402


def device_solve(grid, t, b, m, cfg):
    """Session solve with T resident in HBM; returns q, sd, steps, ms, trace_ms."""
    n = grid.nx * grid.ny * grid.nz
    dev = torch.device("cuda", 0)
    td = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
    q = torch.empty(n, dtype=torch.float64, device=dev)
    sd = torch.empty_like(q)
    s = capi.Session(grid, b, m, cfg)
    s.set_field(td.data_ptr(), True, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    steps = s.solve(0, n, q.data_ptr(), sd.data_ptr(), 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tms = s.timings()[0]
    s.close()
    return q.cpu().numpy(), sd.cpu().numpy(), steps, ms, tms


def sample_cells(n, k, seed=5):
    rng = np.random.default_rng(seed)
    return np.unique(rng.choice(n, size=min(n, k), replace=False)).astype(np.int64)


def cpu_check(grid, t, b, m, cfg, q, sd, k):
    cells = sample_cells(grid.nx * grid.ny * grid.nz, k)
    rq, rsd, rsteps, wall = refshim.solve_cells(grid, t, b, m, cfg, cells)
    rep = fp64_report(q[cells], rq, sd[cells], rsd)
    rep.update(cells=int(len(cells)), cpu_steps=int(rsteps.sum()), cpu_wall_s=wall,
               cpu_steps_per_s=float(rsteps.sum()) / wall, cpu_threads=os.cpu_count())
    return rep


def record(out, **kw):
    line = json.dumps(kw)
    print(line, flush=True)
    with open(out, "a") as f:
        f.write(line + "\n")


def base(name, grid, cfg, steps, ms, tms, prec):
    n = grid.nx * grid.ny * grid.nz
    tot = int(np.sum(steps))
    return dict(config=name, grid=[grid.nx, grid.ny, grid.nz], rays=cfg.rays_per_cell,
                precision=prec, n_levels=cfg.n_levels, total_steps=tot,
                steps_per_ray=tot / (n * cfg.rays_per_cell), solve_ms=ms,
                trace_ms=tms[2], sort_ms=tms[1], reduce_ms=tms[3], setup_ms=tms[0],
                steps_per_s=tot / (ms * 1e-3), trace_steps_per_s=tot / (tms[2] * 1e-3))


def c1(out):
    n = 32
    g = capi.make_grid((n, n, n), (1.0 / n,) * 3)
    t = np.full(n ** 3, 1000.0)
    b = capi.make_boundary((capi.WALL, capi.PERIODIC, capi.PERIODIC),
                           [(0.0, 1.0)] * 3, [(0.0, 1.0)] * 3)
    m = capi.model_from_ermc(E.grey_model(1.0, E.make_planck_bands(900.0, 1100.0, 64),
                                          E.make_temp_grid(900.0, 1100.0, 10.0)))
    cfg = capi.config_struct(rays_per_cell=2000, seed=2024)
    q, sd, steps, ms, tms = device_solve(g, t, b, m, cfg)
    mc = q.reshape(n, n * n).mean(axis=1)
    xs = (np.arange(n) + 0.5) / n
    ref = oracle.slab("const", 1000.0, 1.0, (0.0, 1.0), (0.0, 1.0), xs)
    peak = float(np.max(np.abs(ref)))
    record(out, **base("c1 isothermal grey slab 32^3 kappa=1", g, cfg, steps, ms, tms, "fp64"),
           check="transverse mean vs closed-form slab solution",
           max_err_over_peak=float(np.max(np.abs(mc - ref)) / peak), peak=peak)


def channel(out, name, n, model, tau, prec, rays, k_cells, fp64_ref=None):
    g, t, b, m, _ = W.channel_case(n, model, tau)
    cfg = capi.config_struct(rays_per_cell=rays, seed=2024,
                             precision=capi.FP64 if prec == "fp64" else capi.FP32)
    q, sd, steps, ms, tms = device_solve(g, t, b, m, cfg)
    extra = {}
    if prec == "fp64" and k_cells:
        extra["cpu_parity"] = cpu_check(g, t, b, m, cfg, q, sd, k_cells)
    if prec == "fp32" and fp64_ref is not None:
        fq, fsd = fp64_ref
        bad = three_sigma_violations(q, fq, sd, fsd)
        extra["vs_fp64_same_rays"] = dict(violations_3sigma=bad, allowed=allowed_3sigma(q.size),
                                          max_rel=float(np.max(np.abs(q - fq)) /
                                                        np.max(np.abs(fq))))
    extra["sigma_max"] = float(np.max(sd))
    extra["sigma_median"] = float(np.median(sd))
    record(out, **base(name, g, cfg, steps, ms, tms, prec), **extra)
    return q, sd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "configs.jsonl"))
    ap.add_argument("--only", default="c1,c2,c3,full,fullmg,c4,c5,mg")
    ap.add_argument("--mg-levels", default="1,2,3,4,5,6,7")
    ap.add_argument("--mg-precisions", default="fp64,fp32")
    ap.add_argument("--no-cpu-check", action="store_true",
                    help="skip the multigrid CPU parity samples (timing A/Bs)")
    ap.add_argument("--cells", type=int, default=20000)
    a = ap.parse_args()
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    which = set(a.only.split(","))
    if "c1" in which:
        c1(a.out)
    if "c2" in which:
        for tau in (0.1, 0.3, 1.0, 3.0, 10.0):
            channel(a.out, f"c2 grey channel 128^3 tau={tau}", 128, "grey", tau, "fp64", 64,
                    a.cells // 4)
    if "c3" in which:
        for nb in (16, 119):
            ref = channel(a.out, f"c3 non-grey channel 128^3 {nb}x16", 128, f"nongrey{nb}", 1.0,
                          "fp64", 64, a.cells // 4)
            channel(a.out, f"c3 non-grey channel 128^3 {nb}x16", 128, f"nongrey{nb}", 1.0,
                    "fp32", 64, 0, fp64_ref=ref)
    if "full" in which:
        # Whole-field parity: a config-3 solve (128^3, 16 x 16, R = 64) against
        # the reference's own solve() of the same field on all host threads.
        g, t, b, m, _ = W.channel_case(128, "nongrey16")
        cfg = capi.config_struct(rays_per_cell=64, seed=2024, workers=os.cpu_count() or 1)
        q, sd, steps, ms, tms = device_solve(g, t, b, m, cfg)
        rq, rsd, rsteps, rtotal, rwall = refshim.solve(g, t, b, m, cfg)
        rep = fp64_report(q, rq, sd, rsd)
        rep.update(cpu_total_steps=rtotal, cpu_wall_s=rwall, cpu_steps_per_s=rtotal / rwall,
                   cpu_threads=os.cpu_count(), gpu_total_steps=int(np.sum(steps)),
                   steps_equal=bool(int(np.sum(steps)) == rtotal))
        record(a.out, **base("full-field c3 128^3 16x16 vs reference solve()", g, cfg, steps, ms,
                             tms, "fp64"), full_field_parity=rep)
    if "fullmg" in which:
        # The same whole-field check for multigrid ray coarsening (4 levels).
        g, t, b, m, _ = W.channel_case(128, "nongrey16")
        cfg = capi.config_struct(rays_per_cell=64, seed=2024, workers=os.cpu_count() or 1,
                                 n_levels=4, steps_per_level=5, coarsen_ratio=2)
        q, sd, steps, ms, tms = device_solve(g, t, b, m, cfg)
        rq, rsd, rsteps, rtotal, rwall = refshim.solve(g, t, b, m, cfg)
        rep = fp64_report(q, rq, sd, rsd)
        rep.update(cpu_total_steps=rtotal, cpu_wall_s=rwall, cpu_steps_per_s=rtotal / rwall,
                   cpu_threads=os.cpu_count(), gpu_total_steps=int(np.sum(steps)),
                   steps_equal=bool(int(np.sum(steps)) == rtotal),
                   steps_per_level_equal=bool([int(x) for x in steps] == [int(x) for x in rsteps]))
        record(a.out, **base("full-field c3 128^3 16x16, 4-level multigrid, vs reference solve()",
                             g, cfg, steps, ms, tms, "fp64"),
               steps_per_level=[int(x) for x in steps], full_field_parity=rep)
    if "c4" in which:
        ref = channel(a.out, "c4 non-grey channel 256^3 16x16", 256, "nongrey16", 1.0, "fp64",
                      64, a.cells)
        channel(a.out, "c4 non-grey channel 256^3 16x16", 256, "nongrey16", 1.0, "fp32", 64, 0,
                fp64_ref=ref)
    if "c5" in which:
        for prec in ("fp64", "fp32"):
            rows = []
            for r in (16, 32, 64, 128, 256, 1024):
                g, t, b, m, _ = W.channel_case(256, "nongrey16")
                cfg = capi.config_struct(rays_per_cell=r, seed=7,
                                         precision=capi.FP64 if prec == "fp64" else capi.FP32)
                q, sd, steps, ms, tms = device_solve(g, t, b, m, cfg)
                rows.append((r, float(np.max(sd)), float(np.median(sd)), ms))
                rep = dict(sigma_max=rows[-1][1], sigma_median=rows[-1][2])
                if prec == "fp64" and r in (16, 64):
                    rep["cpu_parity"] = cpu_check(g, t, b, m, cfg, q, sd, a.cells // 4)
                record(a.out, **base(f"c5 rays sweep 256^3 R={r}", g, cfg, steps, ms, tms, prec),
                       **rep)
            lr = np.log([x[0] for x in rows])
            record(a.out, config=f"c5 slopes {prec}",
                   sigma_max_slope=float(np.polyfit(lr, np.log([x[1] for x in rows]), 1)[0]),
                   sigma_median_slope=float(np.polyfit(lr, np.log([x[2] for x in rows]), 1)[0]),
                   time_slope=float(np.polyfit(lr, np.log([x[3] for x in rows]), 1)[0]))
    if "mg" in which:
        g, t, b, m, _ = W.channel_case(256, "nongrey16")
        for prec in a.mg_precisions.split(","):
            for lv in (int(x) for x in a.mg_levels.split(",")):
                cfg = capi.config_struct(rays_per_cell=64, seed=2024, n_levels=lv,
                                         steps_per_level=5, coarsen_ratio=2,
                                         precision=capi.FP64 if prec == "fp64" else capi.FP32)
                q, sd, steps, ms, tms = device_solve(g, t, b, m, cfg)
                rep = {}
                if prec == "fp64" and lv > 1 and not a.no_cpu_check:
                    rep["cpu_parity"] = cpu_check(g, t, b, m, cfg, q, sd, a.cells // 4)
                record(a.out, **base(f"mg multigrid 256^3 levels={lv}", g, cfg, steps, ms, tms,
                                     prec),
                       steps_per_level=[int(x) for x in steps], sigma_max=float(np.max(sd)),
                       sigma_median=float(np.median(sd)), **rep)


if __name__ == "__main__":
    main()
