"""The Python drop-in: `paper_1810_00188_b200` (our `_ermc`) against the
reference's own `_ermc` module (oracle/_ref, built from its unmodified
bindings.cpp) on objects built by the same calls on both sides.

* `solve` (reference proj/python/bindings.cpp:145-147): same q_r / std_dev
  to the fp64 contract, same step counters;
* `solve_numpy` (zero-copy numpy in / out): the same bytes as `solve`;
* the module-level names a reference user imports resolve on ours.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1810_00188_b200 as E
import refshim
from helpers import assert_fp64_parity
from paper_1810_00188_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _build(M, n, model, rays, seed, levels=1):
    """The config-3 channel at n^3 through module M's public API only."""
    g = M.CartesianGrid()
    g.nx = g.ny = g.nz = n
    g.dx, g.dy, g.dz = W.spacing(n)
    f = M.TemperatureField()
    f.grid = g
    f.values = W.channel_field(n).tolist()
    b = M.BoundarySpec()
    b.kind = [M.AxisKind.periodic, M.AxisKind.wall, M.AxisKind.periodic]
    b.lo = [M.Wall(0.0, 1.0), M.Wall(W.T_WALL_LO, 1.0), M.Wall(0.0, 1.0)]
    b.hi = [M.Wall(0.0, 1.0), M.Wall(W.T_WALL_HI, 0.8), M.Wall(0.0, 1.0)]
    temps = M.make_temp_grid(*W.TEMP_GRID)
    if model == "grey":
        m = M.grey_model(0.5, M.make_planck_bands(450.0, 1050.0, 16), temps)
    else:
        sp = M.elsasser_spectrum(temps)
        nu = sp.nu_grid
        m = M.build_k_distribution(sp, M.make_bands(nu[0], nu[-1] + 1e-6, 12),
                                   M.QuadratureSet.gauss_legendre(8))
    c = M.SolveConfig()
    c.rays_per_cell = rays
    c.seed = seed
    c.n_levels = levels
    c.steps_per_level = 4
    return g, f, b, m, c


@pytest.mark.parametrize("model,levels", [("nongrey", 1), ("grey", 1), ("nongrey", 3)])
def test_solve_matches_the_reference_module(model, levels):
    R = refshim.ref_module()
    ref = R.solve(*_build(R, 12, model, 24, 17, levels))
    ours = E.solve(*_build(E, 12, model, 24, 17, levels))
    assert list(ours.steps_per_level) == list(ref.steps_per_level)
    assert ours.total_steps == ref.total_steps
    assert ours.wall_time > 0.0
    assert_fp64_parity(np.array(ours.q_r), np.array(ref.q_r), np.array(ours.std_dev),
                       np.array(ref.std_dev))


def test_solve_numpy_is_solve_without_list_conversion():
    g, f, b, m, c = _build(E, 16, "nongrey", 16, 5)
    sol = E.solve(g, f, b, m, c)
    t = np.asarray(f.values)
    q, sd, steps, total, wall = E.solve_numpy(g, t, b, m, c)
    assert isinstance(q, np.ndarray) and q.dtype == np.float64 and q.shape == (16 ** 3,)
    assert np.array_equal(q, np.array(sol.q_r)) and np.array_equal(sd, np.array(sol.std_dev))
    assert list(steps) == list(sol.steps_per_level) and total == sol.total_steps
    # float32 input is accepted (forcecast) and solved as its float64 values
    q32, *_ = E.solve_numpy(g, t.astype(np.float32), b, m, c)
    q64, *_ = E.solve_numpy(g, t.astype(np.float32).astype(np.float64), b, m, c)
    assert np.array_equal(q32, q64)
    with pytest.raises(RuntimeError, match="does not match the grid"):
        E.solve_numpy(g, t[:-1], b, m, c)


def test_reference_module_names_resolve_on_the_drop_in():
    R = refshim.ref_module()
    solve_path = ["CartesianGrid", "TemperatureField", "BoundarySpec", "Wall", "AxisKind",
                  "NarrowBand", "QuadratureSet", "LineSpectrum", "SpectralModel",
                  "SolveConfig", "SolutionField", "planck_intensity", "make_bands",
                  "make_planck_bands", "make_temp_grid", "grey_model",
                  "build_k_distribution", "elsasser_spectrum", "solve", "lbl_reference",
                  "write_ktab", "read_ktab", "write_tfld", "read_tfld", "write_qrf",
                  "read_qrf", "file_hash"]
    for name in solve_path:
        assert hasattr(R, name), name
        assert hasattr(E, name), name
