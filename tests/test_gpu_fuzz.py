"""Randomised parity: many small random problems, GPU fp64 vs the reference.

Each case draws a grid (odd and even sizes, anisotropic spacing, offset
origin), a boundary (every axis periodic or walled, hot/cold/0 K walls,
emissivity 0..1), a temperature field (smooth + noise), a spectral model
(grey or correlated-k, uniform or non-uniform temperature nodes) and a
configuration (rays, tolerance, step cap, volume sampling, specular walls,
multigrid levels) — so every tracer variant (black-wall, position-tracking,
micro-brick, multigrid, single-node) and dispatch path is exercised against
the reference's own solve() with the fp64 parity contract.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1810_00188_b200 as E
import refshim
from helpers import assert_fp64_parity
from paper_1810_00188_b200 import capi

pytestmark = pytest.mark.gpu


def _case(rng):
    n = [int(rng.integers(2, 12)) for _ in range(3)]
    d = [float(rng.uniform(0.05, 0.3)) for _ in range(3)]
    origin = [float(rng.uniform(-1, 1)) for _ in range(3)]
    g = capi.make_grid(n, d, origin)
    t_lo, t_hi = 500.0, 1500.0
    kind = [int(rng.integers(0, 2)) for _ in range(3)]
    walls = []
    for _ in range(6):
        t = float(rng.choice([0.0, rng.uniform(t_lo, t_hi)]))
        e = float(rng.choice([1.0, 0.0, rng.uniform(0.05, 1.0)]))
        walls.append((t, e))
    b = capi.make_boundary(kind, walls[:3], walls[3:])
    xs = [np.arange(k) / max(k - 1, 1) for k in n]
    base = (800.0 + 300.0 * np.sin(3 * xs[0])[:, None, None] *
            np.cos(2 * xs[1])[None, :, None] + 100.0 * xs[2][None, None, :])
    t = np.clip(base + rng.normal(0, 40, size=base.shape), 550.0, 1450.0).ravel()
    r_err = rng.random()
    if r_err < 0.06:  # invalid inputs: both sides must reject them identically
        t[int(rng.integers(0, t.size))] = float(rng.choice([1600.0, 400.0, -5.0]))
    if rng.random() < 0.5:
        temps = E.make_temp_grid(t_lo, t_hi, float(rng.choice([25.0, 50.0, 100.0])))
    else:  # non-uniform nodes
        temps = sorted({float(x) for x in np.linspace(t_lo, t_hi, 9)} |
                       {float(x) for x in rng.uniform(t_lo, t_hi, 4)})
    if rng.random() < 0.4:
        m = E.grey_model(float(rng.uniform(0.2, 5.0)), E.make_planck_bands(t_lo, t_hi, 8), temps)
    else:
        sp = E.elsasser_spectrum(temps, nu_lo=300.0, nu_hi=2000.0, resolution=2.0,
                                 strength=float(rng.uniform(5.0, 60.0)))
        m = E.build_k_distribution(sp, E.make_bands(sp.nu_grid[0], sp.nu_grid[-1] + 1e-6,
                                                    int(rng.integers(2, 9))),
                                   E.QuadratureSet.gauss_legendre(int(rng.integers(1, 6))))
    levels = int(rng.choice([1, 1, 2, 3]))
    levels = min(levels, 1 + int(np.floor(np.log2(max(n)))))
    cfg = capi.config_struct(
        rays_per_cell=int(rng.integers(1, 33)), seed=int(rng.integers(0, 2**31)),
        tolerance=float(rng.choice([1e-4, 1e-3, 1e-6])),
        max_steps=int(rng.choice([100000, 50, 7])),
        volume_sampling=int(rng.random() < 0.3), specular_walls=int(rng.random() < 0.3),
        n_levels=levels, steps_per_level=int(rng.integers(1, 6)),
        precision=capi.FP64)
    return g, t, b, capi.model_from_ermc(m), cfg


@pytest.mark.parametrize("seed", list(range(64)))
def test_random_problem_matches_reference(seed):
    rng = np.random.default_rng(1000 + seed)
    g, t, b, m, cfg = _case(rng)
    try:
        r = refshim.solve(g, t, b, m, cfg)
    except refshim.RefError as exc:  # the reference rejects it: so must we, verbatim
        with pytest.raises(capi.ErmcError) as info:
            capi.solve(g, t, b, m, cfg)
        assert str(info.value) == str(exc)
        return
    q, sd, steps, total, _ = capi.solve(g, t, b, m, cfg)
    assert total == r[3] and list(steps) == list(r[2])
    assert_fp64_parity(q, r[0], sd, r[1])
