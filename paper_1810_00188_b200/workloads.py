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

import math
import random

import numpy as np

from . import capi

LX, LY, LZ = 4.0 * math.pi, 2.0, 2.0 * math.pi
T_WALL_LO, T_WALL_HI = 955.0, 573.0


def channel_modes(n_modes: int = 24, seed: int = 1234):
    rng = random.Random(seed)
    modes = []
    for _ in range(n_modes):
        kx = rng.randint(1, 6)
        ky = rng.randint(1, 4)
        kz = rng.randint(1, 6)
        phi = rng.uniform(0.0, 2.0 * math.pi)
        a = rng.gauss(0.0, 1.0)
        modes.append((kx, ky, kz, phi, a))
    return modes


def channel_grid(n: int) -> capi.Grid:
    return capi.make_grid((n, n, n), (LX / n, LY / n, LZ / n))


def channel_field(n: int) -> np.ndarray:
    """T at cell centres, k-fastest (i = x, j = y, k = z), float64."""
    dx, dy, dz = LX / n, LY / n, LZ / n
    x = (np.arange(n) + 0.5) * dx
    y = (np.arange(n) + 0.5) * dy
    z = (np.arange(n) + 0.5) * dz
    pert = np.zeros((n, n, n))
    for kx, ky, kz, phi, a in channel_modes():
        cxz = np.cos(kx * x[:, None] / 2.0 + kz * z[None, :] + phi)  # (x, z)
        sy = np.sin(ky * math.pi * y / 2.0)                          # (y,)
        pert += a * cxz[:, None, :] * sy[None, :, None]
    t = (955.0 - 191.0 * y)[None, :, None] + \
        (40.0 / math.sqrt(24.0)) * np.sin(math.pi * y / 2.0)[None, :, None] * pert
    return np.ascontiguousarray(t.reshape(-1))


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
