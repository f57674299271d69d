"""Synthetic workloads of BASELINE.json, built through the
solver's own API so the CPU reference and the GPU consume identical bytes.

* Channel geometry (paper DNS box): N^3 cells over
  Lx = 4 pi (streamwise, periodic), Ly = 2 (wall-normal), Lz = 2 pi
  (spanwise, periodic); walls y_lo = 955 K, y_hi = 573 K, both black.
* Synthetic turbulent temperature:
    T = 955 - 191 y + 40 sin(pi y / 2) / sqrt(24)
          * sum_{m<24} a_m cos(kx_m x / 2 + kz_m z + phi_m) sin(ky_m pi y / 2)
  with random.Random(1234) drawing, per mode in this order, kx in U{1..6},
  ky in U{1..4}, kz in U{1..6}, phi in U(0, 2 pi), a in N(0, 1).
* Grey channel (config 2): grey_model(tau / 2, make_planck_bands(450, 1050, 64),
  make_temp_grid(450, 1050, 5)).
* Non-grey "H2O-like" correlated-k (configs 3-5): elsasser_spectrum with the
  reference defaults on make_temp_grid(450, 1050, 5) ->
  build_k_distribution(make_bands(nu0, nu1 + 1e-6, n_bands),
  gauss_legendre(16)); n_bands = 16 (nb-parab) or 119 (paper H2O count).
"""
from __future__ import annotations

from . import capi
from .channel import (LX, LY, LZ, N_QUAD, T_WALL_HI, T_WALL_LO, TEMP_GRID,  # noqa: F401
                      channel_field, channel_modes, spacing, stratified_runs)


def channel_grid(n: int) -> capi.Grid:
    return capi.make_grid((n, n, n), spacing(n))


def channel_boundary(wall_eps: float = 1.0) -> capi.Boundary:
    """Paper channel walls (black by default; grey walls reflect diffusely)."""
    return capi.make_boundary((capi.PERIODIC, capi.WALL, capi.PERIODIC),
                              [(0.0, 1.0), (T_WALL_LO, wall_eps), (0.0, 1.0)],
                              [(0.0, 1.0), (T_WALL_HI, wall_eps), (0.0, 1.0)])


def _ermc():
    from . import _ermc  # noqa: PLC0415
    return _ermc


def grey_channel_model(tau: float):
    E = _ermc()
    return E.grey_model(tau / 2.0, E.make_planck_bands(450.0, 1050.0, 64),
                        E.make_temp_grid(450.0, 1050.0, 5.0))


def nongrey_channel_model(n_bands: int = 16, n_quad: int = 16, strength: float = 30.0):
    E = _ermc()
    temps = E.make_temp_grid(450.0, 1050.0, 5.0)
    sp = E.elsasser_spectrum(temps, strength=strength)
    return E.build_k_distribution(sp, E.make_bands(sp.nu_grid[0], sp.nu_grid[-1] + 1e-6,
                                                   n_bands),
                                  E.QuadratureSet.gauss_legendre(n_quad))


def file_hashes(n: int, t, model_obj) -> dict:
    """FNV-1a hashes (reference io.cpp:374-389) of the workload's TFLD1 field
    and KTAB1 tables as written by this package's own writers; bench.py's
    reference arm writes the same files with the reference's writers and
    reports the same keys, so equal configs mean byte-identical inputs."""
    import os  # noqa: PLC0415
    import tempfile  # noqa: PLC0415

    E = _ermc()
    g = E.CartesianGrid()
    g.nx = g.ny = g.nz = n
    g.dx, g.dy, g.dz = spacing(n)
    f = E.TemperatureField()
    f.grid = g
    f.values = t.tolist()
    with tempfile.TemporaryDirectory() as d:
        E.write_tfld(os.path.join(d, "t.tfld"), f)
        E.write_ktab(os.path.join(d, "m.ktab"), model_obj)
        return {"tfld_fnv": E.file_hash(os.path.join(d, "t.tfld")),
                "ktab_fnv": E.file_hash(os.path.join(d, "m.ktab"))}


def channel_case(n: int, model: str = "nongrey16", tau: float = 1.0, wall_eps: float = 1.0):
    """(grid, T, boundary, ModelArrays, model_object) for a channel config."""
    if model.startswith("nongrey"):
        nb = int(model[len("nongrey"):] or 16)
        m = nongrey_channel_model(nb)
    elif model == "grey":
        m = grey_channel_model(tau)
    else:
        raise ValueError(model)
    return (channel_grid(n), channel_field(n), channel_boundary(wall_eps),
            capi.model_from_ermc(m), m)
