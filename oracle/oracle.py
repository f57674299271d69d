"""TEST INFRASTRUCTURE ONLY — ctypes access to the C restatement
(oracle/ermc_oracle.c -> oracle/liboracle.so). Only tests/, smoke() and
bench.py's CPU baseline may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
ROOT = HERE.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_1810_00188_b200.capi import Boundary, Config, Grid, Model, RayResult  # noqa: E402

_d = C.POINTER(C.c_double)
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(HERE), "oracle"], check=True,
                           capture_output=True)
        L = C.CDLL(str(LIB))
        L.oracle_uniform.restype = C.c_double
        L.oracle_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]
        L.oracle_build_cdfs.restype = C.c_int
        L.oracle_build_cdfs.argtypes = [C.POINTER(Model), C.c_double, _d, _d, C.c_char_p,
                                        C.c_size_t]
        L.oracle_planck_mean.restype = C.c_int
        L.oracle_planck_mean.argtypes = [C.POINTER(Model), C.c_double, _d, C.c_char_p,
                                         C.c_size_t]
        L.oracle_solve.restype = C.c_int
        L.oracle_solve.argtypes = [C.POINTER(Grid), _d, C.POINTER(Boundary), C.POINTER(Model),
                                   C.POINTER(Config), C.c_int64, C.c_int64, _d, _d,
                                   C.POINTER(C.c_int64), C.c_int, C.c_char_p, C.c_size_t]
        L.oracle_trace_rays.restype = C.c_int
        L.oracle_trace_rays.argtypes = [C.POINTER(Grid), _d, C.POINTER(Boundary),
                                        C.POINTER(Model), C.POINTER(Config), C.c_double,
                                        C.c_double, C.c_int64, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_uint32), _d, C.POINTER(RayResult),
                                        C.c_char_p, C.c_size_t]
        L.oracle_slab.restype = C.c_int
        L.oracle_slab.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_double, _d, C.c_int, C.c_int,
                                  _d, C.c_char_p, C.c_size_t]
        L.oracle_expm1_lean_max_ulp.restype = C.c_double
        L.oracle_expm1_lean_max_ulp.argtypes = [C.c_long, C.POINTER(C.c_long)]
        for f in ("oracle_expint_e1", "oracle_expint_e2", "oracle_expint_e3",
                  "oracle_expm1_lean"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [C.c_double]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def _check(rc, buf):
    if rc:
        raise OracleError(buf.value.decode(errors="replace"))


PROFILES = {"const": 0, "lin1": 1, "lin2": 2, "parab": 3}


def uniform(seed, cell, ray, draw):
    return lib().oracle_uniform(seed, cell, ray, draw)


def build_cdfs(model, t_max):
    band = np.zeros(model.n_bands)
    quad = np.zeros(model.n_bands * model.n_quad)
    buf = C.create_string_buffer(1024)
    _check(lib().oracle_build_cdfs(C.byref(model.desc), t_max, _p(band), _p(quad), buf,
                                   len(buf)), buf)
    return band, quad.reshape(model.n_bands, model.n_quad)


def planck_mean(model, t):
    out = C.c_double()
    buf = C.create_string_buffer(1024)
    _check(lib().oracle_planck_mean(C.byref(model.desc), t, C.byref(out), buf, len(buf)), buf)
    return out.value


def solve(grid, temperature, boundary, model, config, cell_range=None, threads=None):
    """Returns (q_r, std_dev, steps_per_level, total_steps)."""
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    n = grid.nx * grid.ny * grid.nz
    lo, hi = cell_range or (0, n)
    q, sd = np.zeros(hi - lo), np.zeros(hi - lo)
    steps = np.zeros(config.n_levels, dtype=np.int64)
    buf = C.create_string_buffer(1024)
    _check(lib().oracle_solve(C.byref(grid), _p(t), C.byref(boundary), C.byref(model.desc),
                              C.byref(config), lo, hi, _p(q), _p(sd), _p(steps, C.c_int64),
                              threads or os.cpu_count() or 1, buf, len(buf)), buf)
    return q, sd, steps, int(steps.sum())


def trace_rays(grid, temperature, boundary, model, config, t_max, qe, cells, rays, dirs=None):
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    rays = np.ascontiguousarray(rays, dtype=np.uint32)
    out = (RayResult * len(cells))()
    dptr = None
    if dirs is not None:
        dirs = np.ascontiguousarray(dirs, dtype=np.float64).ravel()
        dptr = _p(dirs)
    buf = C.create_string_buffer(1024)
    _check(lib().oracle_trace_rays(C.byref(grid), _p(t), C.byref(boundary),
                                   C.byref(model.desc), C.byref(config), t_max, qe,
                                   len(cells), _p(cells, C.c_int64), _p(rays, C.c_uint32),
                                   dptr, out, buf, len(buf)), buf)
    return list(out)


def slab(profile, t_const, kappa, wall_lo, wall_hi, xs, length=1.0, refine=1):
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    q = np.zeros(len(xs))
    buf = C.create_string_buffer(1024)
    _check(lib().oracle_slab(length, PROFILES[profile], t_const, kappa, wall_lo[0], wall_lo[1],
                             wall_hi[0], wall_hi[1], _p(xs), len(xs), refine, _p(q), buf,
                             len(buf)), buf)
    return q


def expint(order, x):
    return getattr(lib(), f"oracle_expint_e{order}")(x)


def expm1_lean_max_ulp(n):
    d = C.c_long()
    return lib().oracle_expm1_lean_max_ulp(n, C.byref(d)), d.value
