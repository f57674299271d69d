"""Known-answer tests of the device init_ray + march, restating the
reference's tracer/sampling unit tests (proj/tests/test_tracer.cpp,
test_sampling.cpp) through the C-ABI test hook ermc_b200_trace_rays, and
cross-checking every ray against the reference library.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1810_00188_b200 as E
import refshim
from paper_1810_00188_b200 import capi

pytestmark = pytest.mark.gpu

PER = (capi.PERIODIC,) * 3
WALLS = (capi.WALL,) * 3


def wide_grey(kappa):
    # test_tracer.cpp:14-17
    return capi.model_from_ermc(E.grey_model(kappa, E.make_planck_bands(500.0, 1500.0, 32),
                                             E.make_temp_grid(500.0, 1500.0, 50.0)))


def walls(t, eps):
    return capi.make_boundary(WALLS, [(t, eps)] * 3, [(t, eps)] * 3)


def periodic():
    return capi.make_boundary(PER, [(0.0, 1.0)] * 3, [(0.0, 1.0)] * 3)


def both(grid, field, bnd, model, cfg, t_max, qe, cells, rays, dirs=None):
    g, gl = capi.trace_rays(grid, field, bnd, model, cfg, t_max, qe, cells, rays, dirs)
    r, rl = refshim.trace_rays(grid, field, bnd, model, cfg, t_max, qe, cells, rays, dirs)
    for a, b in zip(g, r):
        assert a.steps == b.steps
        assert a.terminated_by == b.terminated_by
        assert a.reflections == b.reflections
        assert (a.band, a.quad, a.next_draw) == (b.band, b.quad, b.next_draw)
        assert a.q_contribution == pytest.approx(b.q_contribution, rel=1e-12, abs=1e-300)
        assert a.prefactor == pytest.approx(b.prefactor, rel=1e-15)
    assert np.array_equal(gl, rl)
    return g, gl


def test_two_cell_hand_computed_exchange():
    # test_tracer.cpp:54-83
    grid = capi.make_grid((2, 1, 1), (1.0, 1.0, 1.0))
    t1, t2 = 800.0, 1200.0
    field = np.array([t1, t2])
    model = wide_grey(1.0)
    mo = E.grey_model(1.0, E.make_planck_bands(500.0, 1500.0, 32),
                      E.make_temp_grid(500.0, 1500.0, 50.0))
    cfg = capi.config_struct(seed=1)
    qe = 100.0
    (res,), _ = both(grid, field, walls(0.0, 1.0), model, cfg, t2, qe, [0], [0],
                     dirs=[1.0, 0.0, 0.0])
    ib1 = mo.interp_ib(res.band, t1)
    ib2 = mo.interp_ib(res.band, t2)
    a1 = 1.0 - math.exp(-0.5)
    a2 = 1.0 - math.exp(-1.0)
    tau1 = 1.0 - a1
    expect = qe * res.prefactor * (tau1 * a2 * (ib2 - ib1) / ib1 +
                                   tau1 * (1.0 - a2) * (0.0 - ib1) / ib1)
    assert res.q_contribution == pytest.approx(expect, rel=1e-9)
    assert res.steps == 2
    assert res.terminated_by == 1  # wall_absorbed


def test_isothermal_rays_exchange_exactly_zero():
    # test_tracer.cpp:38-52
    grid = capi.make_grid((6, 6, 6), (1 / 6,) * 3)
    field = np.full(216, 1000.0)
    cfg = capi.config_struct(seed=4)
    cell = (2 * 6 + 3) * 6 + 1
    res, _ = both(grid, field, walls(1000.0, 1.0), wide_grey(1.0), cfg, 1000.0, 100.0,
                  [cell] * 500, np.arange(500))
    assert all(r.q_contribution == 0.0 for r in res)


def test_black_and_mirror_walls():
    # test_tracer.cpp:85-113
    grid = capi.make_grid((4, 4, 4), (0.25,) * 3)
    field = np.full(64, 900.0)
    cell = (2 * 4 + 2) * 4 + 2
    (r,), _ = both(grid, field, walls(600.0, 1.0), wide_grey(0.1), capi.config_struct(seed=2),
                   900.0, 1.0, [cell], [0])
    assert r.terminated_by == 1 and r.reflections == 0 and r.weight_walls > 0.0
    cell = (1 * 4 + 2) * 4 + 2
    (r,), _ = both(grid, field, walls(600.0, 0.0), wide_grey(1.0), capi.config_struct(seed=2),
                   900.0, 1.0, [cell], [1])
    assert r.terminated_by == 0 and r.reflections > 0 and r.weight_walls == 0.0


@pytest.mark.parametrize("specular", [0, 1])
def test_grey_walls_reflect(specular):
    # test_tracer.cpp:115-131
    grid = capi.make_grid((4, 4, 4), (0.25,) * 3)
    field = np.full(64, 900.0)
    cell = (1 * 4 + 2) * 4 + 2
    cfg = capi.config_struct(seed=5, specular_walls=specular)
    (r,), _ = both(grid, field, walls(700.0, 0.3), wide_grey(1.0), cfg, 900.0, 1.0, [cell], [7])
    assert r.reflections > 0 and r.weight_walls > 0.0


def test_weight_bookkeeping():
    # test_tracer.cpp:133-159
    grid = capi.make_grid((5, 4, 3), (0.2, 0.25, 1.0 / 3))
    field = np.array([700.0 + 50.0 * (c % 7) for c in range(60)])
    bnd = capi.make_boundary((capi.WALL, capi.PERIODIC, capi.WALL),
                             [(600.0, 0.4), (0.0, 1.0), (650.0, 0.7)],
                             [(900.0, 1.0), (0.0, 1.0), (650.0, 0.7)])
    cell = (2 * 4 + 1) * 3 + 1
    res, _ = both(grid, field, bnd, wide_grey(0.8), capi.config_struct(seed=8), 1050.0, 1.0,
                  [cell] * 300, np.arange(300))
    for r in res:
        assert abs(r.weight_absorbed + r.weight_walls + r.weight_residual - 1.0) < 1e-12


def test_residual_below_tolerance_in_periodic_domain():
    # test_tracer.cpp:161-180
    grid = capi.make_grid((4, 4, 4), (0.25,) * 3)
    field = np.full(64, 900.0)
    cell = (1 * 4 + 1) * 4 + 1
    res, _ = both(grid, field, periodic(), wide_grey(2.0), capi.config_struct(seed=3), 900.0,
                  1.0, [cell] * 100, np.arange(100))
    for r in res:
        assert r.terminated_by == 0
        assert 0.0 <= r.weight_residual <= 1e-4


def test_step_cap():
    # test_tracer.cpp:182-198
    grid = capi.make_grid((4, 4, 4), (0.25,) * 3)
    field = np.full(64, 900.0)
    cell = (1 * 4 + 1) * 4 + 1
    cfg = capi.config_struct(seed=3, max_steps=1000)
    (r,), _ = both(grid, field, periodic(), wide_grey(1e-12), cfg, 900.0, 1.0, [cell], [0])
    assert r.terminated_by == 2 and r.steps == 1000


def test_uncapped_multilevel_equals_single_level_bitwise():
    # test_tracer.cpp:200-219
    grid = capi.make_grid((8, 8, 8), (0.125,) * 3)
    field = np.array([700.0 + (c % 11) * 30.0 for c in range(512)])
    cell = (4 * 8 + 4) * 8 + 4
    model = wide_grey(1.0)
    single, _ = capi.trace_rays(grid, field, walls(700.0, 1.0), model,
                                capi.config_struct(seed=6), 1000.0, 10.0, [cell] * 200,
                                np.arange(200))
    multi, _ = both(grid, field, walls(700.0, 1.0), model,
                    capi.config_struct(seed=6, n_levels=3, steps_per_level=2**31 - 1),
                    1000.0, 10.0, [cell] * 200, np.arange(200))
    for a, b in zip(single, multi):
        assert a.q_contribution == b.q_contribution and a.steps == b.steps


def test_demotion_moves_to_coarser_levels():
    # test_tracer.cpp:221-242
    grid = capi.make_grid((16, 16, 16), (1 / 16,) * 3)
    field = np.full(4096, 900.0)
    cell = (8 * 16 + 8) * 16 + 8
    cfg = capi.config_struct(seed=2, n_levels=3, steps_per_level=4)
    res, lvl = both(grid, field, periodic(), wide_grey(0.5), cfg, 900.0, 1.0, [cell] * 50,
                    np.arange(50))
    assert np.all(lvl[:, 0] <= 5)
    assert lvl[:, 2].sum() > 0
    assert np.array_equal(lvl.sum(axis=1), np.array([r.steps for r in res]))


def test_init_ray_draw_order_and_prefactor():
    # test_sampling.cpp:140-191: hottest cell R_I = 1, next_draw 4 / 7.
    grid = capi.make_grid((4, 4, 4), (0.25,) * 3)
    field = np.full(64, 600.0)
    hot = (1 * 4 + 1) * 4 + 1
    field[hot] = 1200.0
    model = capi.model_from_ermc(E.grey_model(2.0, E.make_planck_bands(500.0, 1500.0, 32),
                                              E.make_temp_grid(500.0, 1500.0, 50.0)))
    (r,), _ = both(grid, field, walls(600.0, 1.0), model, capi.config_struct(seed=9), 1200.0,
                   1.0, [hot], [0])
    assert r.prefactor == pytest.approx(1.0, rel=1e-12) and r.next_draw >= 4
    cfg = capi.config_struct(seed=9, volume_sampling=1, specular_walls=1)
    (r,), _ = both(grid, field, walls(600.0, 1.0), model, cfg, 1200.0, 1.0,
                   [(2 * 4 + 1) * 4 + 0], [4])
    assert r.next_draw == 7
    # direction = sample_direction(draw 0, draw 1)
    cid = (1 * 4 + 2) * 4 + 3
    (r,), _ = both(grid, field, walls(600.0, 1.0), model, capi.config_struct(seed=77), 1200.0,
                   1.0, [cid], [5])
    u0, u1 = refshim.uniform(77, cid, 5, 0), refshim.uniform(77, cid, 5, 1)
    ct = 1.0 - 2.0 * u0
    st = math.sqrt(max(0.0, 1.0 - ct * ct))
    assert r.dir[2] == ct
    assert r.dir[0] == pytest.approx(st * math.cos(2 * math.pi * u1), rel=1e-15, abs=1e-300)
