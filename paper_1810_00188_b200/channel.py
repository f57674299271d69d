"""Synthetic turbulent channel temperature field, numpy only.

Kept free of the package's compiled extension so that the reference arm of
bench.py can load it by path and build the exact same T field next to the
reference's own `_ermc` module without mapping any of this repository's
shared libraries.

* Channel geometry (paper DNS box): N^3 cells over
  Lx = 4 pi (streamwise, periodic), Ly = 2 (wall-normal), Lz = 2 pi
  (spanwise, periodic); walls y_lo = 955 K, y_hi = 573 K.
* T = 955 - 191 y + 40 sin(pi y / 2) / sqrt(24)
        * sum_{m<24} a_m cos(kx_m x / 2 + kz_m z + phi_m) sin(ky_m pi y / 2)
  with random.Random(1234) drawing, per mode in this order, kx in U{1..6},
  ky in U{1..4}, kz in U{1..6}, phi in U(0, 2 pi), a in N(0, 1).
"""
from __future__ import annotations

import math
import random

import numpy as np

LX, LY, LZ = 4.0 * math.pi, 2.0, 2.0 * math.pi
T_WALL_LO, T_WALL_HI = 955.0, 573.0
# Correlated-k tables of configs 3-5: elsasser_spectrum (reference defaults,
# spectral.hpp:139-148) on make_temp_grid(450, 1050, 5), n_bands uniform
# bands over its nu grid, gauss_legendre(16).
TEMP_GRID = (450.0, 1050.0, 5.0)
N_QUAD = 16


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


def spacing(n: int):
    return LX / n, LY / n, LZ / n


def channel_field(n: int) -> np.ndarray:
    """T at cell centres, k-fastest (i = x, j = y, k = z), float64."""
    dx, dy, dz = spacing(n)
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


def stratified_runs(n: int, n_runs: int = 256, run: int = 16, seed: int = 5):
    """Parity sample of an n^3 channel: `n_runs` runs of `run` consecutive
    cells along z (k-fastest, so each run is one contiguous cell range), run
    r on wall-normal plane j = r * n // n_runs — every wall distance is
    covered when n_runs >= n — at a random (i, k0). Returns (lo, hi) pairs."""
    rng = np.random.default_rng(seed)
    run = min(run, n)
    out = []
    for r in range(n_runs):
        j = (r * n) // n_runs
        i = int(rng.integers(0, n))
        k0 = int(rng.integers(0, n - run + 1))
        lo = (i * n + j) * n + k0
        out.append((lo, lo + run))
    return sorted(set(out))
