"""TEST INFRASTRUCTURE ONLY — headline (config 4) parity of a GPU solve.

Checks a whole-field GPU solve of a channel workload against the reference
CPU solver on a stratified cell sample, the way SURVEY.md §8c prescribes for
256^3 (a full CPU solve would take minutes): the sampled cells are replayed
through the reference's public build_cdfs / planck_mean / build_hierarchy /
init_ray / march API (oracle/ref_shim.cpp `ref_solve_cells_ex`, the loop of
/root/reference/proj/src/solver.cpp:118-156 — bitwise `solve()` for those
cells), and

  * q_r, std_dev of every sampled cell of the GPU's whole-field solve must
    meet the fp64 contract of tests/helpers.py (1e-9 relative, every cell
    within 3 sigma, sigma to 1e-6);
  * the sample is `n_runs` runs of consecutive cells (one run per
    wall-normal plane); the GPU re-solves each run as its own cell range and
    its march-step count must equal the reference's for that run — step
    parity at a granularity of `run` cells, plus the slab-split invariance
    (the run's q_r / sigma from the range solve must be byte-identical to
    the whole-field solve's).

Used by tests/test_gpu_headline.py and by bench.py (the `parity` block of the
N = 1 line). Never part of the product path.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
for p in (HERE, HERE.parent / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

import refshim  # noqa: E402
from helpers import fp64_report  # noqa: E402


def sample_cells(runs):
    return np.concatenate([np.arange(lo, hi, dtype=np.int64) for lo, hi in runs])


def check(grid, t, b, m, cfg, q_full, sd_full, range_solve, runs, threads=None):
    """range_solve(lo, hi) -> (q[hi-lo], sd[hi-lo], total_steps) on the GPU.

    Returns a dict report; `ok` is the verdict."""
    cells = sample_cells(runs)
    t0 = time.perf_counter()
    rq, rsd, _, cell_steps, cpu_wall = refshim.solve_cells_steps(grid, t, b, m, cfg, cells,
                                                                 threads=threads)
    cpu_s = time.perf_counter() - t0
    rep = fp64_report(np.asarray(q_full)[cells], rq, np.asarray(sd_full)[cells], rsd)
    steps_equal = 0
    split_identical = 0
    off = 0
    for lo, hi in runs:
        q, sd, st = range_solve(lo, hi)
        ref_steps = int(cell_steps[off:off + (hi - lo)].sum())
        steps_equal += int(st == ref_steps)
        split_identical += int(np.array_equal(q, np.asarray(q_full)[lo:hi]) and
                               np.array_equal(sd, np.asarray(sd_full)[lo:hi]))
        off += hi - lo
    out = {
        "cells": int(cells.size), "runs": len(runs), "run_cells": int(runs[0][1] - runs[0][0]),
        "max_rel": rep["max_rel"], "frac_within_1e-9": rep["frac_within_tol"],
        "all_within_3sigma": rep["all_within_3sigma"], "frac_sigma_ok": rep["frac_sd_ok"],
        "bitwise_cells": rep["bitwise_cells"],
        "run_steps_equal": steps_equal, "sample_steps": int(cell_steps.sum()),
        "range_solves_bitwise": split_identical,
        "cpu_reference_s": round(cpu_s, 3), "cpu_trace_s": round(cpu_wall, 3),
        "oracle": "oracle/_ref (unmodified reference) cell-subset replay of solver.cpp:118-156",
    }
    out["ok"] = bool(rep["frac_within_tol"] >= 0.9999 and rep["all_within_3sigma"]
                     and rep["frac_sd_ok"] >= 0.9999 and steps_equal == len(runs)
                     and split_identical == len(runs))
    return out


def torch_range_solver(sess, stream=0, device=0):
    """range_solve for a capi.Session whose field is already set."""
    import torch  # noqa: PLC0415

    dev = torch.device("cuda", device)

    def solve(lo, hi):
        q = torch.empty(hi - lo, dtype=torch.float64, device=dev)
        sd = torch.empty_like(q)
        st = sess.solve(lo, hi, q.data_ptr(), sd.data_ptr(), stream)
        torch.cuda.synchronize(dev)
        return q.cpu().numpy(), sd.cpu().numpy(), int(np.sum(st))
    return solve
