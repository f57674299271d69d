"""Shared helpers for the parity tests: tolerance checks and case builders.

Tolerances:
  fp64 path — per cell |dq| <= 1e-9 * max(|q_ref|, 1e-6 * peak) for at least
  99.99 % of cells and every cell within 3 sigma_ref; sigma relative 1e-6 on
  the same cells; total steps equal (SURVEY §8c recommended criteria).
  fp32 path — |dq| <= 3 sqrt(sigma_a^2 + sigma_b^2) per cell with at most
  0.3 % + 3 sqrt(0.003 N) violators; total steps within 1e-3.
"""
from __future__ import annotations

import math

import numpy as np

REL_FP64 = 1e-9


def fp64_report(q, q_ref, sd, sd_ref):
    q, q_ref, sd, sd_ref = map(np.asarray, (q, q_ref, sd, sd_ref))
    peak = float(np.max(np.abs(q_ref))) if q_ref.size else 0.0
    scale = np.maximum(np.abs(q_ref), 1e-6 * peak)
    dq = np.abs(q - q_ref)
    ok = dq <= REL_FP64 * scale + 0.0
    if peak == 0.0:
        ok = dq == 0.0
    within3 = dq <= 3.0 * sd_ref + (peak * 1e-12)
    sd_scale = np.maximum(np.abs(sd_ref), 1e-6 * max(float(np.max(sd_ref)) if sd_ref.size else 0.0, 0.0))
    sd_ok = np.abs(sd - sd_ref) <= 1e-6 * sd_scale + 0.0
    if sd_ref.size and float(np.max(sd_ref)) == 0.0:
        sd_ok = np.abs(sd - sd_ref) == 0.0
    rel = dq / np.where(scale > 0, scale, 1.0)
    return {
        "n": int(q.size),
        "peak": peak,
        "frac_within_tol": float(np.mean(ok)) if q.size else 1.0,
        "all_within_3sigma": bool(np.all(within3)),
        "frac_sd_ok": float(np.mean(sd_ok)) if q.size else 1.0,
        "max_rel": float(np.max(rel)) if q.size else 0.0,
        "bitwise_cells": int(np.sum(q == q_ref)),
    }


def assert_fp64_parity(q, q_ref, sd, sd_ref, min_frac=0.9999):
    r = fp64_report(q, q_ref, sd, sd_ref)
    assert r["frac_within_tol"] >= min_frac, r
    assert r["all_within_3sigma"], r
    assert r["frac_sd_ok"] >= min_frac, r
    return r


def three_sigma_violations(qa, qb, sda, sdb):
    qa, qb, sda, sdb = map(np.asarray, (qa, qb, sda, sdb))
    sig = np.sqrt(sda * sda + sdb * sdb)
    bad = np.abs(qa - qb) > 3.0 * sig
    both_zero = (sig == 0) & (qa == qb)
    return int(np.sum(bad & ~both_zero))


def allowed_3sigma(n: int) -> int:
    return int(0.003 * n + 3.0 * math.sqrt(0.003 * n) + 1)


# ---- golden fixtures -------------------------------------------------------
from pathlib import Path as _Path  # noqa: E402

GOLDEN = _Path(__file__).resolve().parent / "golden"
CONFIG_KEYS = ["rays_per_cell", "n_levels", "tolerance", "seed", "max_steps", "sorting",
               "steps_per_level", "coarsen_ratio", "volume_sampling", "specular_walls"]


def golden_names():
    return sorted(p.stem[len("solve_"):] for p in GOLDEN.glob("solve_*.npz"))


def load_model(z):
    from paper_1810_00188_b200 import capi
    return capi.ModelArrays(z["m_nu_lo"], z["m_nu_hi"], z["m_nu_center"], z["m_g"], z["m_w"],
                            z["m_temps"], z["m_k"], z["m_ib"])


def load_golden_solve(name):
    """(grid, T, boundary, model, config, expected dict) of a golden solve."""
    from paper_1810_00188_b200 import capi
    z = np.load(GOLDEN / f"solve_{name}.npz")
    grid = capi.make_grid(z["grid_n"], z["grid_d"], z["grid_origin"])
    b = capi.make_boundary(z["b_kind"], list(zip(z["b_lo_t"], z["b_lo_e"])),
                           list(zip(z["b_hi_t"], z["b_hi_e"])))
    cfg_vals = dict(zip(CONFIG_KEYS, z["config"].tolist()))
    ints = {k: int(v) for k, v in cfg_vals.items() if k != "tolerance"}
    cfg = capi.config_struct(tolerance=cfg_vals["tolerance"], **ints)
    expected = dict(q_r=z["q_r"], std_dev=z["std_dev"], steps=z["steps_per_level"],
                    total=int(z["total_steps"][0]))
    return grid, z["temperature"], b, load_model(z), cfg, expected
