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
                   slabs are assembled on every rank (the reduction kernel
                   storing into peers' buffers over CUDA IPC, or NCCL).
                   `e2e`: the C-ABI call ermc_b200_solve_range with pinned
                   host buffers (H2D of T, D2H of Q_r / sigma inside the timed
                   region). N = 1 adds `parity` (the timed solve's field vs
                   the reference CPU solver on 4096 stratified cells),
                   `roofline.l2` (measured L2 bandwidth) and `cpu_baseline`
                   (the reference arm below, run as a subprocess).
  --impl reference the UNMODIFIED reference through its own public API: the
                   `_ermc` pybind module compiled from /root/reference's
                   sources into oracle/_ref, inputs built with its own
                   builders (elsasser_spectrum, build_k_distribution, ...),
                   each step one stock `solve()` over the whole field at
                   --ref-rays rays per cell (a bounded sample of the R-ray
                   workload: every cell, ray ids 0..ref_rays-1), workers =
                   the host threads available; rank 0 only. This process
                   never maps a shared library of this repository's package.

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py launches
the N ranks itself (127.0.0.1 rendezvous, the same env torchrun sets).
"""
from __future__ import annotations

import argparse
import json
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
    p.add_argument("--ref-rays", type=int, default=1,
                   help="rays per cell of each reference-arm sample solve (whole field)")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-single-worker", action="store_true")
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
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        pw = [num(r[2]) for r in rows if num(r[2]) is not None]
        load = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        busy = [p for p in pw if p > 0.5 * (max(pw) if pw else 1)]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        capped = sum(1 for r in rows if r[7] == "Active")
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "sw_power_cap_samples": capped,
                "power_w_median": statistics.median(busy) if busy else None,
                "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------- shared
def config_dict(a, world, hashes):
    """The `config` of both arms (identical dicts = the same workload on
    byte-identical inputs: the FNV-1a hashes of the TFLD1 field and KTAB1
    tables each arm wrote with its own writers)."""
    return {"workload": workload_name(a), "grid": a.grid, "rays_per_cell": a.rays,
            "model": a.model, "precision": a.precision, "seed": a.seed,
            "parallelism": f"x-slabs x{world} (cells split in contiguous ranges; "
                           "the reference's worker chunks)",
            "l2": "flushed (256 MiB write) before every GPU step",
            "tfld_fnv": hashes.get("tfld_fnv"), "ktab_fnv": hashes.get("ktab_fnv")}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_by_path(name, path):
    import importlib.util  # noqa: PLC0415

    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ----------------------------------------------------------------- reference arm
class ReferenceSolver:
    """The reference's own `_ermc` module (oracle/_ref: its bindings.cpp and
    src/*.cpp compiled unmodified by oracle/Makefile) and the workload built
    through its own API. Loads nothing from paper_1810_00188_b200/ except the
    numpy-only channel.py (by path, not as a package import)."""

    def __init__(self, a):
        ref_dir = ROOT / "oracle" / "_ref"
        if not list(ref_dir.glob("_ermc*.so")):
            raise FileNotFoundError("oracle/_ref/_ermc is not built (make -C oracle ref)")
        sys.path.insert(0, str(ref_dir))
        import _ermc as E  # noqa: PLC0415  (the reference's module)

        sys.path.pop(0)
        if "oracle/_ref" not in str(Path(E.__file__).resolve()):
            raise RuntimeError(f"wrong _ermc module loaded: {E.__file__}")
        self.E = E
        ch = load_by_path("ermc_channel", ROOT / "paper_1810_00188_b200" / "channel.py")
        n = a.grid
        g = E.CartesianGrid()
        g.nx = g.ny = g.nz = n
        g.dx, g.dy, g.dz = ch.spacing(n)
        f = E.TemperatureField()
        f.grid = g
        f.values = ch.channel_field(n).tolist()
        b = E.BoundarySpec()
        b.kind = [E.AxisKind.periodic, E.AxisKind.wall, E.AxisKind.periodic]
        b.lo = [E.Wall(0.0, 1.0), E.Wall(ch.T_WALL_LO, a.wall_eps), E.Wall(0.0, 1.0)]
        b.hi = [E.Wall(0.0, 1.0), E.Wall(ch.T_WALL_HI, a.wall_eps), E.Wall(0.0, 1.0)]
        temps = E.make_temp_grid(*ch.TEMP_GRID)
        if a.model.startswith("nongrey"):
            nb = int(a.model[len("nongrey"):] or 16)
            sp = E.elsasser_spectrum(temps)  # ElsasserParams{} defaults (strength 30)
            nu = sp.nu_grid
            m = E.build_k_distribution(sp, E.make_bands(nu[0], nu[-1] + 1e-6, nb),
                                       E.QuadratureSet.gauss_legendre(ch.N_QUAD))
        elif a.model == "grey":
            m = E.grey_model(0.5, E.make_planck_bands(450.0, 1050.0, 64), temps)
        else:
            raise ValueError(a.model)
        self.grid, self.field, self.boundary, self.model = g, f, b, m
        import tempfile  # noqa: PLC0415

        with tempfile.TemporaryDirectory() as d:
            E.write_tfld(os.path.join(d, "t.tfld"), f)
            E.write_ktab(os.path.join(d, "m.ktab"), m)
            self.hashes = {"tfld_fnv": E.file_hash(os.path.join(d, "t.tfld")),
                           "ktab_fnv": E.file_hash(os.path.join(d, "m.ktab"))}
        self.seed = a.seed

    def solve(self, rays, workers, field=None, grid=None):
        c = self.E.SolveConfig()
        c.rays_per_cell = rays
        c.seed = self.seed
        c.workers = workers
        return self.E.solve(grid or self.grid, field or self.field, self.boundary, self.model, c)

    def single_worker(self, n=128):
        """Per-core rate: stock solve with workers = 1 on the same channel at
        n^3 (the 256^3 field at one worker would take minutes), R = 1."""
        E = self.E
        ch = load_by_path("ermc_channel", ROOT / "paper_1810_00188_b200" / "channel.py")
        g = E.CartesianGrid()
        g.nx = g.ny = g.nz = n
        g.dx, g.dy, g.dz = ch.spacing(n)
        f = E.TemperatureField()
        f.grid = g
        f.values = ch.channel_field(n).tolist()
        s = self.solve(1, 1, field=f, grid=g)
        return {"value": s.total_steps / s.wall_time, "unit": UNIT, "workers": 1,
                "sample": f"stock solve(), workers=1, {n}^3 channel, R=1 "
                          f"({s.total_steps} steps in {s.wall_time:.1f} s)"}


def run_reference(a, world, rank):
    if rank != 0:
        return
    threads = host_threads()
    ref = ReferenceSolver(a)
    n_cells = a.grid ** 3
    vals, walls, steps_l = [], [], []
    for i in range(a.warmup + a.steps):
        s = ref.solve(a.ref_rays, threads)
        if i >= a.warmup:
            vals.append(s.total_steps / s.wall_time)
            walls.append(s.wall_time)
            steps_l.append(s.total_steps)
    value = sum(steps_l) / sum(walls)
    steps_per_ray = steps_l[-1] / (n_cells * a.ref_rays)
    steps_field = steps_per_ray * n_cells * a.rays
    sample = (f"stock ermc::solve() of the reference's own _ermc module over all {n_cells} "
              f"cells at R={a.ref_rays} (ray ids 0..{a.ref_rays - 1} of the workload's "
              f"R={a.rays}; {steps_l[-1]} steps in {walls[-1]:.2f} s per step), "
              f"workers={threads}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (turbulent channel T field + Elsasser correlated-k tables, "
                "built with the reference's own builders)",
        "config": config_dict(a, world, ref.hashes),
        "s_per_field_extrapolated": steps_field / value,
        "steps_per_ray": steps_per_ray,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model(),
                         "threads_visible": host_threads(), "cpu_count": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if not a.no_single_worker:
        try:
            line["cpu_baseline"]["single_worker"] = ref.single_worker()
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"]["single_worker"] = {"error": str(exc)}
    print(json.dumps(line), flush=True)


def cpu_baseline_subprocess(a):
    """The reference arm (one sample step, no warm-up) in a child process, so
    the GPU arm's process never loads the reference module and vice versa."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
           "--warmup", "0", "--grid", str(a.grid), "--rays", str(a.rays), "--model", a.model,
           "--seed", str(a.seed), "--wall-eps", str(a.wall_eps), "--precision", a.precision,
           "--ref-rays", str(a.ref_rays)]
    if a.no_single_worker:
        cmd.append("--no-single-worker")
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
        for line in r.stdout.splitlines():
            if line.startswith("{"):
                d = json.loads(line)
                cb = d["cpu_baseline"]
                cb["config_hashes"] = {k: d["config"].get(k) for k in ("tfld_fnv", "ktab_fnv")}
                return cb
        return {"error": (r.stderr or r.stdout)[-500:]}
    except Exception as exc:  # pragma: no cover
        return {"error": str(exc)}


# ----------------------------------------------------------------- GPU arm
def run_b200(a, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_1810_00188_b200 import capi, parallel, workloads as W

    n_dev = max(1, torch.cuda.device_count())
    # Ranks sharing a GPU (more ranks than devices: the one-GPU test box)
    # cannot use NCCL (one communicator rank per device); they use gloo, the
    # collectives go through host memory and the timings mean nothing. The
    # driver's runs use NCCL, one GPU per rank. ERMC_BENCH_BACKEND overrides.
    shared = world > n_dev
    backend = os.environ.get("ERMC_BENCH_BACKEND", "gloo" if shared else "nccl")
    local = local % n_dev
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            # the communicator's INIT lines (nranks, NVLS / P2P transports)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # collective tensors
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    grid, t_host, b, m, m_obj = W.channel_case(a.grid, a.model, wall_eps=a.wall_eps)
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
    # the solve. "nccl": all-gather of the slabs (gloo when ranks share a
    # GPU). ERMC_BENCH_GATHER overrides; if the IPC mappings cannot be made
    # the run falls back to the all-gather and says so.
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
            gather, outs = "all-gather (fused unavailable)", None
    elif gather == "nccl":
        gather = "all-gather"

    def device_resident(precision, steps, warmup, keep=False):
        cfg = capi.config_struct(rays_per_cell=a.rays, seed=a.seed, precision=precision,
                                 device=local)
        sess = capi.Session(grid, b, m, cfg)
        sess.set_field(t_dev.data_ptr(), True, sptr)
        q = torch.empty(slab.n, dtype=torch.float64, device=dev)
        sd = torch.empty_like(q)
        trace_ms, launches, total_steps = 0.0, 0, 0
        full = [None]

        def one():
            flush.zero_()
            if outs is not None:  # reduction writes every rank's full field
                return sess.solve_scatter(slab.lo, slab.hi, outs[0], outs[1], sptr)
            st = sess.solve(slab.lo, slab.hi, q.data_ptr(), sd.data_ptr(), sptr)
            if world > 1:
                full[0] = (parallel.gather_slabs(q, slabs, dist),
                           parallel.gather_slabs(sd, slabs, dist))
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
        if keep:
            return elapsed, trace_ms, launches, total_steps, sess, q, sd
        sess.close()
        return elapsed, trace_ms, launches, total_steps

    clocks = ClockSampler(local)
    clocks.start()
    keep = world == 1 and rank == 0 and not a.no_parity and a.precision == "fp64"
    res = device_resident(prec, a.steps, a.warmup, keep=keep)
    clk = clocks.stop()
    el, trace_ms, launches, local_steps = res[:4]
    el_max = max_over_ranks(el)
    all_steps = sum_over_ranks(local_steps)
    value = all_steps / (el_max * 1e-3)
    steps_per_field = all_steps / a.steps
    peak, peak_kind = peaks()
    bps = BYTES_PER_STEP[a.precision]
    trace_s = trace_ms * 1e-3
    achieved = local_steps * bps / trace_s / 1e9  # GB/s of the trace kernel
    # Per-step DRAM and L2 traffic of the committed `ncu --set full` capture
    # (profiles/ncu_trace_summary.json, same kernel, 256^3 channel) times the
    # steps of one launch here.
    traffic, l2 = None, None
    prof = ROOT / "profiles" / "ncu_trace_summary.json"
    pj = {}
    if prof.exists():
        try:
            pj = json.loads(prof.read_text()).get(a.precision, {})
        except Exception:
            pj = {}
    if "dram_bytes_per_step" in pj:
        traffic = pj["dram_bytes_per_step"] * local_steps / a.steps
    try:
        l2_peak = capi.probe_l2(local, 48 << 20, 20, 0)
        l2_gather = capi.probe_l2(local, 48 << 20, 4, 1)
        l2 = {"peak": l2_peak, "unit": "GB/s",
              "peak_source": "measured: ermc_b200_probe_l2 streaming 16-B ld.global.cg over "
                             "a 48 MiB L2-resident buffer",
              "gather_peak": l2_gather,
              "gather_source": "measured: independent hashed 8-B loads, 32-B sectors counted"}
        if "l2_bytes_per_step" in pj:
            l2_ach = pj["l2_bytes_per_step"] * local_steps / trace_s / 1e9
            l2.update(achieved=l2_ach, frac=l2_ach / l2_peak,
                      bytes_per_step=pj["l2_bytes_per_step"],
                      bytes_source=f"ncu lts__t_bytes / steps of capture {pj.get('capture')}",
                      ncu_lts_throughput_pct=pj.get("lts_throughput_pct"))
    except Exception as exc:  # pragma: no cover
        l2 = {"error": str(exc)}

    parity = None
    if keep:
        sess, q, sd = res[4], res[5], res[6]
        try:
            sys.path[:0] = [str(ROOT / "oracle"), str(ROOT / "tests")]
            import headline  # noqa: PLC0415  (test infrastructure: the checker)

            cfg = capi.config_struct(rays_per_cell=a.rays, seed=a.seed)
            parity = headline.check(grid, t_host, b, m, cfg, q.cpu().numpy(), sd.cpu().numpy(),
                                    headline.torch_range_solver(sess, sptr, local),
                                    W.stratified_runs(a.grid, 256, 16))
            parity["solve"] = "the last timed step's field (fp64)"
        except Exception as exc:  # pragma: no cover
            parity = {"ok": False, "error": str(exc)}
        finally:
            sess.close()

    extra = {}
    if not a.no_fp32_extra and a.precision == "fp64":
        el32, tr32, nl32, st32 = device_resident(capi.FP32, a.steps, 1)
        el32 = max_over_ranks(el32)
        s32 = sum_over_ranks(st32)
        ach32 = st32 * BYTES_PER_STEP["fp32"] / (tr32 * 1e-3) / 1e9
        extra["fp32"] = {"value": s32 / (el32 * 1e-3), "unit": UNIT, "dtype": "f32",
                         "s_per_field": el32 * 1e-3 / a.steps,
                         "parity": "statistical (3 sigma vs the reference, "
                                   "tests/test_gpu_headline.py), same rays",
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

    hashes = W.file_hashes(a.grid, t_host, m_obj) if rank == 0 else {}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline_subprocess(a)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": el_max / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if a.precision == "fp64" else "f32",
            "data": "synthetic (turbulent channel T field + Elsasser correlated-k tables, "
                    "generated through the solver API)",
            "config": config_dict(a, world, hashes),
            "gather": gather if world > 1 else None,
            "backend": backend if world > 1 else None,
            "ranks_share_gpu": shared if world > 1 else None,
            "s_per_field": el_max * 1e-3 / a.steps,
            "steps_per_field": steps_per_field,
            "steps_per_ray": steps_per_field / (n_cells * a.rays),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{peak_kind} hbm_gbs",
                         "bytes_per_step": bps, "kernel": f"trace_pool_{a.precision}",
                         "kernel_ms_per_step": trace_ms / a.steps,
                         "traffic_source": "ncu dram bytes/step x steps per launch",
                         "l2": l2},
            "parity": parity,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(a):
    """`bench.py --gpus N` without a launcher: start N ranks of this script
    with the environment torchrun would give them (127.0.0.1 rendezvous)."""
    import socket  # noqa: PLC0415

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(a.gpus):
        env = dict(os.environ, WORLD_SIZE=str(a.gpus), RANK=str(r), LOCAL_RANK=str(r),
                   LOCAL_WORLD_SIZE=str(a.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, *sys.argv], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    # A rank that fails would leave the others blocked in a collective: stop
    # them (these are our own children, by PID) and report the failure.
    while True:
        codes = [pr.poll() for pr in procs]
        if any(c not in (None, 0) for c in codes):
            for pr in procs:
                if pr.poll() is None:
                    pr.kill()
            return max(c for c in (pr.wait() for pr in procs) if c is not None) or 1
        if all(c == 0 for c in codes):
            return 0
        time.sleep(0.5)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    world, rank, local = dist_env()
    if world != a.gpus and rank == 0:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}; using {world}\n")
    if a.impl == "reference":
        run_reference(a, world, rank)
    else:
        run_b200(a, world, rank, local)


if __name__ == "__main__":
    main()
