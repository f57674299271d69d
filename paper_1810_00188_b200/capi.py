"""ctypes binding of the C-ABI boundary (include/ermc_b200.h).

This is the FFI stub a reference-side maintainer would add:
plain structs and pointers, no torch or pybind types. Tests and bench.py call
the GPU path through it. Descriptors can be built from numpy arrays or from
`_ermc` objects (`model_from_ermc`, ...).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Sequence

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("ERMC_B200_LIB", _HERE / "libermc_b200.so"))
# ERMC_B200_LIB: load another build of the same library (A/B experiments on
# one GPU box; tools/ab_lib.sh).

PERIODIC, WALL = 0, 1
FP64, FP32 = 0, 1

_d = C.POINTER(C.c_double)


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("reserved0", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
                ("dz", C.c_double), ("origin", C.c_double * 3)]


class Boundary(C.Structure):
    _fields_ = [("kind", C.c_int32 * 3), ("reserved0", C.c_int32),
                ("lo_temperature", C.c_double * 3), ("lo_emissivity", C.c_double * 3),
                ("hi_temperature", C.c_double * 3), ("hi_emissivity", C.c_double * 3)]


class Model(C.Structure):
    _fields_ = [("n_bands", C.c_int32), ("n_quad", C.c_int32), ("n_temps", C.c_int32),
                ("reserved0", C.c_int32), ("band_nu_lo", _d), ("band_nu_hi", _d),
                ("band_nu_center", _d), ("g_points", _d), ("g_weights", _d),
                ("temp_grid", _d), ("k_table", _d), ("ib_table", _d)]


class Config(C.Structure):
    _fields_ = [("rays_per_cell", C.c_int32), ("n_levels", C.c_int32),
                ("tolerance", C.c_double), ("seed", C.c_uint64),
                ("max_steps", C.c_int64), ("sorting", C.c_int32),
                ("steps_per_level", C.c_int32), ("coarsen_ratio", C.c_int32),
                ("volume_sampling", C.c_int32), ("specular_walls", C.c_int32),
                ("workers", C.c_int32), ("precision", C.c_int32), ("device", C.c_int32),
                ("n_devices", C.c_int32), ("reserved0", C.c_int32)]


class Solution(C.Structure):
    _fields_ = [("q_r", _d), ("std_dev", _d), ("steps_per_level", C.POINTER(C.c_int64)),
                ("total_steps", C.c_int64), ("wall_time", C.c_double)]


class RayResult(C.Structure):
    _fields_ = [("q_contribution", C.c_double), ("weight_absorbed", C.c_double),
                ("weight_walls", C.c_double), ("weight_residual", C.c_double),
                ("dir", C.c_double * 3), ("prefactor", C.c_double),
                ("ib_source", C.c_double), ("steps", C.c_int64),
                ("terminated_by", C.c_int32), ("reflections", C.c_int32),
                ("band", C.c_int32), ("quad", C.c_int32), ("next_draw", C.c_uint32),
                ("reserved0", C.c_int32)]


class RayState(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("dir", C.c_double * 3), ("cell", C.c_int32 * 4),
                ("transmissivity", C.c_double), ("band", C.c_int32), ("quad", C.c_int32),
                ("prefactor", C.c_double), ("ib_source", C.c_double),
                ("reflections", C.c_int32), ("reserved0", C.c_int32), ("seed", C.c_uint64),
                ("cell_id", C.c_uint64), ("ray_id", C.c_uint32), ("next_draw", C.c_uint32)]


EXPORTS = {
    "ermc_b200_config_default": (None, [C.POINTER(Config)]),
    "ermc_b200_solve": (C.c_int, [C.POINTER(Grid), _d, C.POINTER(Boundary),
                                  C.POINTER(Model), C.POINTER(Config),
                                  C.POINTER(Solution), C.c_char_p, C.c_size_t]),
    "ermc_b200_solve_range": (C.c_int, [C.POINTER(Grid), _d, C.POINTER(Boundary),
                                        C.POINTER(Model), C.POINTER(Config), C.c_int64,
                                        C.c_int64, C.POINTER(Solution), C.c_char_p,
                                        C.c_size_t]),
    "ermc_b200_session_create": (C.c_void_p, [C.POINTER(Grid), C.POINTER(Boundary),
                                              C.POINTER(Model), C.POINTER(Config),
                                              C.c_char_p, C.c_size_t]),
    "ermc_b200_session_destroy": (None, [C.c_void_p]),
    "ermc_b200_session_set_field": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int,
                                              C.c_void_p, C.c_char_p, C.c_size_t]),
    "ermc_b200_session_solve": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                                          C.c_char_p, C.c_size_t]),
    "ermc_b200_session_timings": (C.c_int, [C.c_void_p, _d, C.POINTER(C.c_int32)]),
    "ermc_b200_session_solve_async": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                                C.c_void_p, C.c_void_p, C.c_char_p,
                                                C.c_size_t]),
    "ermc_b200_session_wait": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.c_char_p,
                                         C.c_size_t]),
    "ermc_b200_session_solve_scatter": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64,
                                                  C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                                  C.c_int32, C.POINTER(C.c_int64), C.c_void_p,
                                                  C.c_char_p, C.c_size_t]),
    "ermc_b200_device_alloc": (C.c_int, [C.c_int, C.c_size_t, C.POINTER(C.c_void_p), C.c_char_p,
                                         C.c_size_t]),
    "ermc_b200_device_free": (C.c_int, [C.c_void_p]),
    "ermc_b200_ipc_export": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_char_p, C.c_size_t]),
    "ermc_b200_ipc_open": (C.c_int, [C.POINTER(C.c_uint8), C.POINTER(C.c_void_p), C.c_char_p,
                                     C.c_size_t]),
    "ermc_b200_ipc_close": (C.c_int, [C.c_void_p]),
    "ermc_b200_trace_rays": (C.c_int, [C.POINTER(Grid), _d, C.POINTER(Boundary),
                                       C.POINTER(Model), C.POINTER(Config), C.c_double,
                                       C.c_double, C.c_int64, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_uint32), _d, C.POINTER(RayResult),
                                       C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]),
    "ermc_b200_sample_direction": (C.c_int, [C.c_int64, _d, _d, _d, C.c_char_p, C.c_size_t]),
    "ermc_b200_absorptivity": (C.c_int, [C.c_int64, _d, _d, _d, C.c_char_p, C.c_size_t]),
    "ermc_b200_init_rays": (C.c_int, [C.POINTER(Grid), _d, C.POINTER(Model), _d, _d, C.c_double,
                                      C.c_uint64, C.c_int32, C.c_int64, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_uint32), C.POINTER(RayState), C.c_char_p,
                                      C.c_size_t]),
    "ermc_b200_march_rays": (C.c_int, [C.c_int32, C.POINTER(Grid), C.POINTER(_d),
                                       C.POINTER(C.c_int32), C.POINTER(Model),
                                       C.POINTER(Boundary), C.c_double, C.c_double, C.c_int64,
                                       C.c_int32, C.c_int64, C.POINTER(RayState),
                                       C.POINTER(RayResult), C.POINTER(C.c_int64), C.c_char_p,
                                       C.c_size_t]),
    "ermc_b200_build_cdfs": (C.c_int, [C.POINTER(Model), C.c_double, _d, _d,
                                       C.c_char_p, C.c_size_t]),
    "ermc_b200_planck_mean": (C.c_int, [C.POINTER(Model), C.c_double, _d, C.c_char_p,
                                        C.c_size_t]),
    "ermc_b200_uniform_device": (C.c_int, [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                           _d, C.c_char_p, C.c_size_t]),
    "ermc_b200_device_count": (C.c_int, []),
    "ermc_b200_abi_version": (C.c_int, []),
    "ermc_b200_release_cached_memory": (C.c_int, [C.c_int]),
    "ermc_b200_probe_l2": (C.c_int, [C.c_int, C.c_size_t, C.c_int, C.c_int, _d, C.c_char_p,
                                     C.c_size_t]),
}


class ErmcError(RuntimeError):
    """Error returned through the C-ABI (the reference's ermc::Error text)."""


_lib = None


def load(path: Path | str = LIB_PATH) -> C.CDLL:
    """Loads libermc_b200.so and declares every exported signature."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not Path(path).exists():
        raise ImportError(f"{path} is missing: build with `python paper_1810_00188_b200/build.py`"
                          " (there is no CPU fallback)")
    lib = C.CDLL(str(path))
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib


def _ptr(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


class ModelArrays:
    """Owns contiguous float64 arrays for an ermc_model_t descriptor."""

    def __init__(self, nu_lo, nu_hi, nu_center, g_points, g_weights, temps, k_table,
                 ib_table):
        f = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())  # noqa: E731
        self.nu_lo, self.nu_hi, self.nu_center = f(nu_lo), f(nu_hi), f(nu_center)
        self.g_points, self.g_weights = f(g_points), f(g_weights)
        self.temps, self.k_table, self.ib_table = f(temps), f(k_table), f(ib_table)
        self.desc = Model(len(self.nu_lo), len(self.g_points), len(self.temps), 0,
                          _ptr(self.nu_lo), _ptr(self.nu_hi), _ptr(self.nu_center),
                          _ptr(self.g_points), _ptr(self.g_weights), _ptr(self.temps),
                          _ptr(self.k_table), _ptr(self.ib_table))

    @property
    def n_bands(self) -> int:
        return len(self.nu_lo)

    @property
    def n_quad(self) -> int:
        return len(self.g_points)


def model_from_ermc(model) -> ModelArrays:
    """Descriptor arrays from an `_ermc.SpectralModel` (either implementation:
    ours exposes the tables as methods; the reference's via its bands())."""
    bands = model.bands()
    q = model.quadrature()
    return ModelArrays([b.nu_lo for b in bands], [b.nu_hi for b in bands],
                       [b.nu_center for b in bands], q.g_points, q.weights,
                       model.temp_grid(), model.k_table(), model.ib_table())


def make_grid(n: Sequence[int], d: Sequence[float], origin=(0.0, 0.0, 0.0)) -> Grid:
    g = Grid()
    g.nx, g.ny, g.nz = (int(v) for v in n)
    g.dx, g.dy, g.dz = (float(v) for v in d)
    for a in range(3):
        g.origin[a] = float(origin[a])
    return g


def make_boundary(kind: Sequence[int], lo: Sequence[tuple], hi: Sequence[tuple]) -> Boundary:
    """kind[a] in {PERIODIC, WALL}; lo/hi[a] = (temperature, emissivity)."""
    b = Boundary()
    for a in range(3):
        b.kind[a] = int(kind[a])
        b.lo_temperature[a], b.lo_emissivity[a] = (float(v) for v in lo[a])
        b.hi_temperature[a], b.hi_emissivity[a] = (float(v) for v in hi[a])
    return b


def make_config(**kw) -> Config:
    c = Config()
    load().ermc_b200_config_default(C.byref(c))
    for k, v in kw.items():
        if not hasattr(c, k):
            raise KeyError(k)
        setattr(c, k, v)
    return c


def default_config_values() -> dict:
    """Reference SolveConfig defaults (solver.hpp:12-26) without loading the
    library (used by CPU tests)."""
    return dict(rays_per_cell=2000, n_levels=1, tolerance=1e-4, seed=0, max_steps=100000,
                sorting=0, steps_per_level=5, coarsen_ratio=2, volume_sampling=0,
                specular_walls=0, workers=0, precision=FP64, device=-1, n_devices=1)


def config_struct(**kw) -> Config:
    """Config from the reference defaults, without touching the library."""
    vals = default_config_values()
    vals.update(kw)
    c = Config()
    for k, v in vals.items():
        setattr(c, k, v)
    return c


def _err() -> C.Array:
    return C.create_string_buffer(2048)


def _raise(rc: int, buf) -> None:
    if rc != 0:
        raise ErmcError(buf.value.decode(errors="replace"))


def solve(grid: Grid, temperature: np.ndarray, boundary: Boundary, model: ModelArrays,
          config: Config, cell_range: tuple[int, int] | None = None):
    """ermc_b200_solve / _solve_range with host buffers.

    Returns (q_r, std_dev, steps_per_level, total_steps, wall_time)."""
    lib = load()
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    n_total = grid.nx * grid.ny * grid.nz
    lo, hi = (0, n_total) if cell_range is None else cell_range
    q = np.zeros(hi - lo)
    sd = np.zeros(hi - lo)
    steps = np.zeros(max(config.n_levels, 1), dtype=np.int64)
    sol = Solution(_ptr(q), _ptr(sd), _ptr(steps, C.c_int64), 0, 0.0)
    buf = _err()
    if cell_range is None:
        rc = lib.ermc_b200_solve(C.byref(grid), _ptr(t), C.byref(boundary),
                                 C.byref(model.desc), C.byref(config), C.byref(sol),
                                 buf, len(buf))
    else:
        rc = lib.ermc_b200_solve_range(C.byref(grid), _ptr(t), C.byref(boundary),
                                       C.byref(model.desc), C.byref(config), lo, hi,
                                       C.byref(sol), buf, len(buf))
    _raise(rc, buf)
    return q, sd, steps, int(sol.total_steps), float(sol.wall_time)


def trace_rays(grid, temperature, boundary, model, config, t_max, q_emission, cells,
               rays, dirs=None):
    """ermc_b200_trace_rays: list of RayResult plus per-level steps array."""
    lib = load()
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    rays = np.ascontiguousarray(rays, dtype=np.uint32)
    n = len(cells)
    out = (RayResult * n)()
    lvl = np.zeros(n * config.n_levels, dtype=np.int64)
    dptr = None
    if dirs is not None:
        dirs = np.ascontiguousarray(dirs, dtype=np.float64).ravel()
        dptr = _ptr(dirs)
    buf = _err()
    rc = lib.ermc_b200_trace_rays(C.byref(grid), _ptr(t), C.byref(boundary),
                                  C.byref(model.desc), C.byref(config), t_max, q_emission,
                                  n, _ptr(cells, C.c_int64), _ptr(rays, C.c_uint32), dptr,
                                  out, _ptr(lvl, C.c_int64), buf, len(buf))
    _raise(rc, buf)
    return list(out), lvl.reshape(n, config.n_levels)


def build_cdfs(model: ModelArrays, t_max: float):
    lib = load()
    band = np.zeros(model.n_bands)
    quad = np.zeros(model.n_bands * model.n_quad)
    buf = _err()
    _raise(lib.ermc_b200_build_cdfs(C.byref(model.desc), t_max, _ptr(band), _ptr(quad),
                                    buf, len(buf)), buf)
    return band, quad.reshape(model.n_bands, model.n_quad)


def planck_mean(model: ModelArrays, t: float) -> float:
    lib = load()
    out = C.c_double()
    buf = _err()
    _raise(lib.ermc_b200_planck_mean(C.byref(model.desc), t, C.byref(out), buf, len(buf)),
           buf)
    return out.value


def device_alloc(device: int, nbytes: int) -> int:
    lib = load()
    p = C.c_void_p()
    buf = _err()
    _raise(lib.ermc_b200_device_alloc(device, nbytes, C.byref(p), buf, len(buf)), buf)
    return p.value


def ipc_export(ptr: int) -> bytes:
    lib = load()
    h = (C.c_uint8 * 64)()
    buf = _err()
    _raise(lib.ermc_b200_ipc_export(C.c_void_p(ptr), h, buf, len(buf)), buf)
    return bytes(h)


def ipc_open(handle: bytes) -> int:
    lib = load()
    h = (C.c_uint8 * 64)(*handle)
    p = C.c_void_p()
    buf = _err()
    _raise(lib.ermc_b200_ipc_open(h, C.byref(p), buf, len(buf)), buf)
    return p.value


def probe_l2(device: int = 0, nbytes: int = 48 << 20, iters: int = 20, mode: int = 0) -> float:
    """Measured L2 read bandwidth, GB/s (mode 0 streaming, 1 sector gather)."""
    lib = load()
    out = C.c_double()
    buf = _err()
    _raise(lib.ermc_b200_probe_l2(device, nbytes, iters, mode, C.byref(out), buf, len(buf)), buf)
    return out.value


def uniform_device(seed: int, cells, rays, draws) -> np.ndarray:
    lib = load()
    cells = np.ascontiguousarray(cells, dtype=np.uint64)
    rays = np.ascontiguousarray(rays, dtype=np.uint32)
    draws = np.ascontiguousarray(draws, dtype=np.uint32)
    out = np.zeros(len(cells))
    buf = _err()
    _raise(lib.ermc_b200_uniform_device(seed, len(cells), _ptr(cells, C.c_uint64),
                                        _ptr(rays, C.c_uint32), _ptr(draws, C.c_uint32),
                                        _ptr(out), buf, len(buf)), buf)
    return out


class Session:
    """Device-resident session (ermc_b200_session_*): the field stays in HBM;
    outputs go to caller-provided device pointers (e.g. torch tensors)."""

    def __init__(self, grid: Grid, boundary: Boundary, model: ModelArrays, config: Config):
        self._lib = load()
        self._keep = (grid, boundary, model, config)
        buf = _err()
        self.h = self._lib.ermc_b200_session_create(C.byref(grid), C.byref(boundary),
                                                    C.byref(model.desc), C.byref(config),
                                                    buf, len(buf))
        if not self.h:
            raise ErmcError(buf.value.decode(errors="replace"))
        self.n_levels = config.n_levels

    def set_field(self, ptr: int, is_device: bool, stream: int = 0) -> None:
        buf = _err()
        _raise(self._lib.ermc_b200_session_set_field(self.h, C.c_void_p(ptr),
                                                     1 if is_device else 0,
                                                     C.c_void_p(stream), buf, len(buf)), buf)

    def solve(self, lo: int, hi: int, d_q: int, d_sd: int, stream: int = 0) -> np.ndarray:
        steps = np.zeros(self.n_levels, dtype=np.int64)
        buf = _err()
        _raise(self._lib.ermc_b200_session_solve(self.h, lo, hi, C.c_void_p(d_q),
                                                 C.c_void_p(d_sd), _ptr(steps, C.c_int64),
                                                 C.c_void_p(stream), buf, len(buf)), buf)
        return steps

    def solve_async(self, lo: int, hi: int, d_q: int, d_sd: int, stream: int = 0) -> None:
        """Enqueue the solve of [lo, hi) on `stream` and return; see wait()."""
        buf = _err()
        _raise(self._lib.ermc_b200_session_solve_async(self.h, lo, hi, C.c_void_p(d_q),
                                                       C.c_void_p(d_sd), C.c_void_p(stream),
                                                       buf, len(buf)), buf)

    def wait(self) -> np.ndarray:
        """Block until the pending solve is done; its per-level step counts."""
        steps = np.zeros(self.n_levels, dtype=np.int64)
        buf = _err()
        _raise(self._lib.ermc_b200_session_wait(self.h, _ptr(steps, C.c_int64), buf, len(buf)),
               buf)
        return steps

    def solve_scatter(self, lo: int, hi: int, q_full: Sequence[int], sd_full: Sequence[int],
                      stream: int = 0) -> np.ndarray:
        """Solve [lo, hi) and store each cell's result into every buffer of
        q_full / sd_full (device pointers: this GPU's and IPC-mapped peers')."""
        steps = np.zeros(self.n_levels, dtype=np.int64)
        n = len(q_full)
        qa = (C.c_void_p * n)(*q_full)
        sa = (C.c_void_p * n)(*sd_full)
        buf = _err()
        _raise(self._lib.ermc_b200_session_solve_scatter(
            self.h, lo, hi, qa, sa, n, _ptr(steps, C.c_int64), C.c_void_p(stream), buf,
            len(buf)), buf)
        return steps

    def timings(self) -> tuple[list[float], int]:
        ms = np.zeros(4)
        n = C.c_int32()
        self._lib.ermc_b200_session_timings(self.h, _ptr(ms), C.byref(n))
        return ms.tolist(), n.value

    def close(self) -> None:
        if self.h:
            self._lib.ermc_b200_session_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
