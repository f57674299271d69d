#!/usr/bin/env python
"""Benchmark of the ERMC Q_r solve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One "step" is one full Q_r field solve of the configured workload (default:
BASELINE config 4 — the 256^3 non-grey correlated-k channel, 16 bands x
16 g-points, R = 64 rays/cell, seed 2024; synthetic T field and tables built
through the solver's own API, see paper_1810_00188_b200/workloads.py).
Metric: ray-cell steps/s over all ranks (= total march iterations /
max-over-ranks device time), plus seconds per Q_r field.

Arms
  default          the B200 path. `value`: inputs resident in HBM (session
                   API, device pointers), timed with CUDA events over exactly
                   K steps between barriers, L2 flushed (256 MiB write) before
                   every step; N > 1 ranks each solve their x-slab and the
                   slabs are all-gathered (NCCL). `e2e`: the C-ABI call
                   ermc_b200_solve_range with pinned host buffers (H2D of T,
                   D2H of Q_r / sigma inside the timed region).
  --impl reference the reference's own CPU solver (oracle/_ref, compiled from
                   the unmodified sources) on the host cores, each step a
                   bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import signal
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "ray-cell steps/s & s per Q_r field, 256³ non-grey, 1/2/4/8 B200 vs host CPU"
UNIT = "ray-cell steps/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
BYTES_PER_STEP = {"fp64": 40.0, "fp32": 20.0}  # SURVEY §8d / BASELINE.md


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--grid", type=int, default=256)
    p.add_argument("--rays", type=int, default=64)
    p.add_argument("--model", default="nongrey16")
    p.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    p.add_argument("--seed", type=int, default=2024)
    p.add_argument("--wall-eps", type=float, default=1.0,
                   help="channel wall emissivity (1 = config 4's black walls)")
    p.add_argument("--no-fp32-extra", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d.get("hbm_gbs", FALLBACK_HBM_GBS)), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def workload_name(a):
    walls = "" if a.wall_eps == 1.0 else f", grey walls eps={a.wall_eps}"
    return (f"config4: {a.grid}^3 synthetic turbulent channel, {a.model} correlated-k "
            f"(elsasser, 16 g), R={a.rays} rays/cell, seed {a.seed}{walls}")


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"ermc_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.send_signal(signal.SIGTERM)
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                rows.append(f)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        load = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------- CPU arm
class CpuReference:
    """The reference solver (oracle/_ref: unmodified sources) on a stratified
    sample of the workload's cells, through the cell-subset replay of
    solver.cpp:118-156 (bitwise the reference's solve() for those cells).
    The timing covers the march loop, not the O(N) per-call setup copies."""

    def __init__(self, grid, t, b, m, cfg, threads):
        sys.path.insert(0, str(ROOT / "oracle"))
        import refshim  # noqa: PLC0415

        self.n = grid.nx * grid.ny * grid.nz
        self.threads = threads
        if refshim.available():
            self.run = lambda cells: refshim.solve_cells(grid, t, b, m, cfg, cells,
                                                         threads=threads)
            self.kind = "reference"
        else:  # the C restatement (port) if the reference could not be built
            import oracle  # noqa: PLC0415

            def run(cells):
                t0 = time.perf_counter()
                lo, hi = int(cells[0]), int(cells[-1]) + 1
                q, sd, st, tot = oracle.solve(grid, t, b, m, cfg, cell_range=(lo, hi),
                                              threads=threads)
                return q, sd, st, time.perf_counter() - t0
            self.run = run
            self.kind = "port"
        self.cells = None

    def size(self, seconds):
        want = max(self.threads * 4, 32)
        while True:
            cells = np.unique(np.linspace(0, self.n - 1, min(self.n, want)).astype(np.int64))
            _, _, st, wall = self.run(cells)
            if wall >= 0.5 * seconds or len(cells) >= self.n:
                break
            want = int(want * min(8.0, max(1.5, 0.9 * seconds / max(wall, 1e-3))))
        self.cells = cells

    def step(self):
        _, _, st, wall = self.run(self.cells)
        steps = int(np.sum(st))
        return steps / wall, steps, wall, len(self.cells)


def cpu_reference_sample(grid, t, b, m, cfg, seconds, threads):
    ref = CpuReference(grid, t, b, m, cfg, threads)
    ref.size(seconds)
    v, steps, wall, n = ref.step()
    return v, steps, wall, n, ref.kind


def run_reference(a, world, rank):
    if rank != 0:
        return
    from paper_1810_00188_b200 import capi, workloads as W

    grid, t, b, m, _ = W.channel_case(a.grid, a.model, wall_eps=a.wall_eps)
    cfg = capi.config_struct(rays_per_cell=a.rays, seed=a.seed, workers=os.cpu_count() or 1)
    threads = os.cpu_count() or 1
    ref = CpuReference(grid, t, b, m, cfg, threads)
    ref.size(max(2.0, min(a.cpu_seconds, 6.0)))  # ~5 s per step: K + W steps stay within minutes
    vals = []
    last = None
    for i in range(a.warmup + a.steps):
        r = ref.step()
        if i >= a.warmup:
            vals.append(r[0])
            last = r + (ref.kind,)
    value = sum(vals) / len(vals)
    n_cells = a.grid ** 3
    sample = (f"{last[3]} stratified cells of {n_cells} x R={a.rays} "
              f"({last[1]} steps in {last[2]:.1f} s) per step")
    spf = a.grid ** 3 * a.rays * (last[1] / (last[3] * a.rays)) / value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": last[2] * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload_name(a), "grid": a.grid,
                                        "rays_per_cell": a.rays, "model": a.model},
        "s_per_field_extrapolated": spf,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": last[4],
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def run_b200(a, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_1810_00188_b200 import capi, parallel, workloads as W

    # ERMC_BENCH_BACKEND=gloo (test only): ranks may share one GPU (device =
    # local rank mod visible devices) and the collectives go through host
    # memory, so the N > 1 flow can be exercised on a one-GPU box. Timings
    # from such a run mean nothing; the driver's runs use NCCL, one GPU each.
    backend = os.environ.get("ERMC_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # collective tensors
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    grid, t_host, b, m, _ = W.channel_case(a.grid, a.model, wall_eps=a.wall_eps)
    n_cells = grid.nx * grid.ny * grid.nz
    slabs = parallel.all_slabs(grid.nx, grid.ny, grid.nz, world)
    slab = slabs[rank]
    prec = capi.FP64 if a.precision == "fp64" else capi.FP32

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        v = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        v = torch.tensor([x], dtype=torch.int64, device=cdev)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        return int(v.item())

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    t_dev = torch.from_numpy(t_host).to(dev)

    # N > 1: how Q_r / sigma are assembled on every rank. "fused" (default):
    # the solve's reduction kernel stores each cell straight into every rank's
    # full-field buffer (CUDA IPC mappings; NVLink stores), no collective after
    # the solve. "nccl": all-gather of the slabs. ERMC_BENCH_GATHER overrides;
    # if the IPC mappings cannot be made the run uses NCCL and says so.
    gather = os.environ.get("ERMC_BENCH_GATHER", "fused") if world > 1 else "none"
    outs = None
    if gather == "fused":
        try:
            q_full = capi.device_alloc(local, n_cells * 8)
            sd_full = capi.device_alloc(local, n_cells * 8)
            handles = [None] * world
            dist.all_gather_object(handles, (capi.ipc_export(q_full), capi.ipc_export(sd_full)))
            outs = ([q_full if r == rank else capi.ipc_open(handles[r][0]) for r in range(world)],
                    [sd_full if r == rank else capi.ipc_open(handles[r][1]) for r in range(world)])
            ok = 1
        except Exception as exc:  # pragma: no cover - depends on the node
            ok = 0
            sys.stderr.write(f"fused gather unavailable: {exc}\n")
        flag = torch.tensor([ok], dtype=torch.int64, device=cdev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            gather, outs = "nccl (fused unavailable)", None

    def device_resident(precision, steps, warmup):
        cfg = capi.config_struct(rays_per_cell=a.rays, seed=a.seed, precision=precision,
                                 device=local)
        sess = capi.Session(grid, b, m, cfg)
        sess.set_field(t_dev.data_ptr(), True, sptr)
        q = torch.empty(slab.n, dtype=torch.float64, device=dev)
        sd = torch.empty_like(q)
        trace_ms, launches, total_steps = 0.0, 0, 0

        def one():
            flush.zero_()
            if outs is not None:  # reduction writes every rank's full field
                return sess.solve_scatter(slab.lo, slab.hi, outs[0], outs[1], sptr)
            st = sess.solve(slab.lo, slab.hi, q.data_ptr(), sd.data_ptr(), sptr)
            if world > 1:
                parallel.gather_slabs(q, slabs, dist)
                parallel.gather_slabs(sd, slabs, dist)
            return st

        for _ in range(warmup):
            one()
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            st = one()
            ms, nl = sess.timings()
            trace_ms += ms[2]
            launches += nl
            total_steps += int(st.sum())
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        elapsed = e0.elapsed_time(e1)
        sess.close()
        return elapsed, trace_ms, launches, total_steps

    clocks = ClockSampler(local)
    clocks.start()
    el, trace_ms, launches, local_steps = device_resident(prec, a.steps, a.warmup)
    clk = clocks.stop()
    el_max = max_over_ranks(el)
    all_steps = sum_over_ranks(local_steps)
    value = all_steps / (el_max * 1e-3)
    steps_per_field = all_steps / a.steps
    peak, peak_kind = peaks()
    bps = BYTES_PER_STEP[a.precision]
    achieved = local_steps * bps / (trace_ms * 1e-3) / 1e9  # GB/s of the trace kernel
    # DRAM traffic per launch: bytes/step of the committed `ncu --set full`
    # capture (profiles/ncu_trace_summary.json, same kernel, 256^3 channel)
    # times the steps of one launch here.
    traffic = None
    prof = ROOT / "profiles" / "ncu_trace_summary.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text()).get(a.precision, {})
            if "dram_bytes_per_step" in pj:
                traffic = pj["dram_bytes_per_step"] * local_steps / a.steps
        except Exception:
            traffic = None

    extra = {}
    if not a.no_fp32_extra and a.precision == "fp64":
        el32, tr32, nl32, st32 = device_resident(capi.FP32, a.steps, 1)
        el32 = max_over_ranks(el32)
        s32 = sum_over_ranks(st32)
        ach32 = st32 * BYTES_PER_STEP["fp32"] / (tr32 * 1e-3) / 1e9
        extra["fp32"] = {"value": s32 / (el32 * 1e-3), "unit": UNIT, "dtype": "f32",
                         "s_per_field": el32 * 1e-3 / a.steps,
                         "parity": "statistical (3 sigma vs fp64), same rays",
                         "roofline": {"bound": "hbm", "achieved": ach32, "peak": peak,
                                      "unit": "GB/s", "frac": ach32 / peak,
                                      "bytes_per_step": BYTES_PER_STEP["fp32"]}}

    e2e = None
    if not a.no_e2e:
        pin_t = torch.from_numpy(t_host).pin_memory()
        q_h = torch.empty(slab.n, dtype=torch.float64).pin_memory()
        sd_h = torch.empty(slab.n, dtype=torch.float64).pin_memory()
        cfg = capi.config_struct(rays_per_cell=a.rays, seed=a.seed, precision=prec, device=local)
        import ctypes as C
        lib = capi.load()
        steps_arr = np.zeros(1, dtype=np.int64)
        sol = capi.Solution(C.cast(q_h.data_ptr(), C.POINTER(C.c_double)),
                            C.cast(sd_h.data_ptr(), C.POINTER(C.c_double)),
                            steps_arr.ctypes.data_as(C.POINTER(C.c_int64)), 0, 0.0)
        buf = C.create_string_buffer(2048)
        tptr = C.cast(pin_t.data_ptr(), C.POINTER(C.c_double))

        def e2e_one():
            rc = lib.ermc_b200_solve_range(C.byref(grid), tptr, C.byref(b), C.byref(m.desc),
                                           C.byref(cfg), slab.lo, slab.hi, C.byref(sol), buf,
                                           len(buf))
            if rc:
                raise RuntimeError(buf.value.decode())
            return sol.total_steps

        e2e_one()
        barrier()
        t0 = time.perf_counter()
        tot = 0
        for _ in range(a.steps):
            tot += e2e_one()
        wall = time.perf_counter() - t0
        barrier()
        wall = max_over_ranks(wall)
        tot = sum_over_ranks(tot)
        e2e = {"value": tot / wall, "unit": UNIT, "h2d_bytes_per_step": n_cells * 8,
               "d2h_bytes_per_step": slab.n * 16, "s_per_field": wall / a.steps,
               "path": "ermc_b200_solve_range (C-ABI), pinned host T in / Q_r, sigma out"}

    cpu = None
    if rank == 0 and world == 1:
        cfg = capi.config_struct(rays_per_cell=a.rays, seed=a.seed, workers=os.cpu_count() or 1)
        threads = os.cpu_count() or 1
        r = cpu_reference_sample(grid, t_host, b, m, cfg, a.cpu_seconds, threads)
        cpu = {"value": r[0], "unit": UNIT, "cores": threads, "kind": r[4],
               "sample": f"{r[3]} stratified cells of {n_cells} x R={a.rays} "
                         f"({r[1]} steps in {r[2]:.1f} s), oracle/_ref solve_cells"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": el_max / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if a.precision == "fp64" else "f32",
            "data": "synthetic (turbulent channel T field + Elsasser correlated-k tables, "
                    "generated through the solver API)",
            "config": {"workload": workload_name(a), "grid": a.grid, "rays_per_cell": a.rays,
                       "model": a.model, "precision": a.precision,
                       "parallelism": f"x-slabs x{world}" + (
                           "" if world == 1 else
                           " + all-gather fused into the reduction (CUDA IPC, NVLink stores)"
                           if gather == "fused" else f" + {backend} all-gather"),
                       "l2": "flushed (256 MiB write) before every step"},
            "s_per_field": el_max * 1e-3 / a.steps,
            "steps_per_field": steps_per_field,
            "steps_per_ray": steps_per_field / (n_cells * a.rays),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{peak_kind} hbm_gbs",
                         "bytes_per_step": bps, "kernel": f"trace_pool_{a.precision}",
                         "kernel_ms_per_step": trace_ms / a.steps,
                         "traffic_source": "ncu dram bytes/step x steps per launch"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    world, rank, local = dist_env()
    if a.impl == "reference":
        run_reference(a, world, rank)
    else:
        run_b200(a, world, rank, local)


if __name__ == "__main__":
    main()
