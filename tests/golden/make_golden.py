"""Generates the golden vectors in tests/golden/ from the REFERENCE itself.

Run in the container (needs oracle/_ref, i.e. `make -C oracle ref`):
    python tests/golden/make_golden.py
Each case stores its complete inputs (grid, T, boundary, model tables,
config) next to the reference's outputs, so tests can replay it without the
reference present. Outputs come from the unmodified reference library:
solve() (proj/src/solver.cpp:82-180), init_ray+march (sampling.cpp:55-96,
tracer.cpp:57-194), build_cdfs/planck_mean (spectral.cpp:207-218,306-354),
uniform (sampling.cpp:24-29) and slab_oracle (oracles.cpp:73-128).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import refshim  # noqa: E402
from paper_1810_00188_b200 import capi  # noqa: E402
from paper_1810_00188_b200 import workloads as W  # noqa: E402

CONFIG_KEYS = ["rays_per_cell", "n_levels", "tolerance", "seed", "max_steps", "sorting",
               "steps_per_level", "coarsen_ratio", "volume_sampling", "specular_walls"]

SOLVES = [
    # name, source, grid_n, config overrides
    ("isothermal_6", "isothermal", 6, dict(rays_per_cell=16, seed=1)),
    ("grey_lin1_8", "grey-lin1", 8, dict(rays_per_cell=16, seed=11)),
    ("grey_parab_8", "grey-parab", 8, dict(rays_per_cell=16, seed=3)),
    ("box_sin_5_6", "box-sin-5", 6, dict(rays_per_cell=8, seed=2)),
    ("epsw_low_6", "epsw-low", 6, dict(rays_per_cell=8, seed=5)),
    ("epsw_low_6_specular", "epsw-low", 6, dict(rays_per_cell=8, seed=5, specular_walls=1)),
    ("epsw_01_6_volume", "epsw-01", 6, dict(rays_per_cell=8, seed=6, volume_sampling=1)),
    ("nb_parab_6", "nb-parab", 6, dict(rays_per_cell=16, seed=7)),
    ("nb_3dimens_6_multigrid", "nb-3dimens", 6, dict(rays_per_cell=8, seed=9, n_levels=3,
                                                    steps_per_level=2)),
    ("grey_parab_8_capped", "grey-parab", 8, dict(rays_per_cell=8, seed=4, max_steps=5)),
    ("channel_nongrey16_8", "channel:nongrey16", 8, dict(rays_per_cell=8, seed=2024)),
    ("channel_grey_tau1_8", "channel:grey", 8, dict(rays_per_cell=8, seed=2024)),
]


def case_inputs(source, n):
    if source.startswith("channel:"):
        g, t, b, m, _ = W.channel_case(n, source.split(":")[1], tau=1.0)
        return g, t, b, m
    g, t, b, m, _ = refshim.ref_case(source, n)
    return g, t, b, m


def pack_inputs(g, t, b, m, cfg):
    return dict(
        grid_n=np.array([g.nx, g.ny, g.nz]), grid_d=np.array([g.dx, g.dy, g.dz]),
        grid_origin=np.array(list(g.origin)), temperature=t,
        b_kind=np.array(list(b.kind)), b_lo_t=np.array(list(b.lo_temperature)),
        b_lo_e=np.array(list(b.lo_emissivity)), b_hi_t=np.array(list(b.hi_temperature)),
        b_hi_e=np.array(list(b.hi_emissivity)), m_nu_lo=m.nu_lo, m_nu_hi=m.nu_hi,
        m_nu_center=m.nu_center, m_g=m.g_points, m_w=m.g_weights, m_temps=m.temps,
        m_k=m.k_table, m_ib=m.ib_table,
        config=np.array([getattr(cfg, k) for k in CONFIG_KEYS], dtype=np.float64))


def main():
    manifest = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref (unmodified "
                "/root/reference/proj/src compiled by oracle/Makefile)", "cases": {}}
    for name, source, n, over in SOLVES:
        g, t, b, m = case_inputs(source, n)
        cfg = capi.config_struct(workers=1, **over)
        q, sd, steps, total, _ = refshim.solve(g, t, b, m, cfg)
        data = pack_inputs(g, t, b, m, cfg)
        data.update(q_r=q, std_dev=sd, steps_per_level=steps, total_steps=np.array([total]))
        np.savez_compressed(HERE / f"solve_{name}.npz", **data)
        manifest["cases"][name] = {"source": source, "grid_n": n, "config": over,
                                   "total_steps": total}
        print(name, total)

    # Keyed RNG (sampling.cpp:24-29): 256 keys incl. large ids.
    rng = np.random.default_rng(2024)
    seeds = rng.integers(0, 2**63, 256, dtype=np.uint64)
    cells = rng.integers(0, 2**40, 256, dtype=np.uint64)
    rays = rng.integers(0, 2**32, 256, dtype=np.uint32)
    draws = rng.integers(0, 200, 256, dtype=np.uint32)
    vals = np.array([refshim.uniform(int(s), int(c), int(r), int(d))
                     for s, c, r, d in zip(seeds, cells, rays, draws)])
    np.savez_compressed(HERE / "uniform.npz", seed=seeds, cell=cells, ray=rays, draw=draws,
                        value=vals)

    # CDFs and Planck means for the channel non-grey model.
    _, _, _, m = case_inputs("channel:nongrey16", 4)
    out = {}
    for tm in (573.0, 800.0, 955.0):
        bc, qc = refshim.build_cdfs(m, tm)
        out[f"band_{tm:g}"] = bc
        out[f"quad_{tm:g}"] = qc
        out[f"kp_{tm:g}"] = np.array([refshim.planck_mean(m, tm)])
    np.savez_compressed(HERE / "cdfs_channel16.npz", m_nu_lo=m.nu_lo, m_nu_hi=m.nu_hi,
                        m_nu_center=m.nu_center, m_g=m.g_points, m_w=m.g_weights,
                        m_temps=m.temps, m_k=m.k_table, m_ib=m.ib_table, **out)

    # Analytic grey slab (config 1 and the paper's grey-slab verification).
    R = refshim.ref_module()
    xs = (np.arange(32) + 0.5) / 32
    slabs = {}
    for key, prof, t_lo, e_lo, t_hi, e_hi in [
            ("iso1000_cold", lambda x: 1000.0, 0.0, 1.0, 0.0, 1.0),
            ("lin1", lambda x: 500.0 + 1000.0 * x, 500.0, 1.0, 1500.0, 1.0),
            ("parab", lambda x: 500.0 - 2000.0 * x * x + 2000.0 * x, 500.0, 1.0, 500.0, 1.0),
            ("lin2_eps01", lambda x: 295.0 + 10.0 * x, 295.0, 0.0, 305.0, 1.0)]:
        sc = R.SlabCase()
        sc.length = 1.0
        sc.t_profile = prof
        sc.kappa = 1.0
        sc.wall_lo = R.Wall(t_lo, e_lo)
        sc.wall_hi = R.Wall(t_hi, e_hi)
        slabs[key] = np.array(R.slab_oracle(sc, list(xs)))
    slabs["x"] = xs
    slabs["e1"] = np.array([R.expint_e1(v) for v in (0.01, 0.5, 1.0, 2.5, 10.0)])
    slabs["e2"] = np.array([R.expint_e2(v) for v in (0.0, 0.01, 0.5, 1.0, 2.5, 10.0)])
    slabs["e3"] = np.array([R.expint_e3(v) for v in (0.0, 0.01, 0.5, 1.0, 2.5, 10.0)])
    np.savez_compressed(HERE / "slab_oracle.npz", **slabs)
    (HERE / "MANIFEST.json").write_text(json.dumps(manifest, indent=1) + "\n")


if __name__ == "__main__":
    main()
