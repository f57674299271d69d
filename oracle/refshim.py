"""TEST INFRASTRUCTURE ONLY — ctypes access to the reference CPU solver.

Loads oracle/_ref/libermc_ref.so (the UNMODIFIED reference sources compiled
by oracle/Makefile, plus ref_shim.cpp) and oracle/_ref/_ermc (the
reference's own pybind module). Both are built in the container from
/root/reference and travel to the GPU box as binaries; nothing here reads
/root/reference at run time.

Only tests/, __graft_entry__.smoke() and bench.py's CPU arms may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
REF_LIB = REF_DIR / "libermc_ref.so"
ROOT = HERE.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_1810_00188_b200 import capi  # noqa: E402  (descriptor layouts only)
from paper_1810_00188_b200.capi import Boundary, Config, Grid, Model, RayResult, Solution  # noqa: E402

_d = C.POINTER(C.c_double)
_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} missing: run `make -C oracle ref` in the container")
        L = C.CDLL(str(REF_LIB))
        L.ref_solve.restype = C.c_int
        L.ref_solve.argtypes = [C.POINTER(Grid), _d, C.POINTER(Boundary), C.POINTER(Model),
                                C.POINTER(Config), C.POINTER(Solution), C.c_char_p, C.c_size_t]
        L.ref_solve_cells.restype = C.c_int
        L.ref_solve_cells.argtypes = [C.POINTER(Grid), _d, C.POINTER(Boundary),
                                      C.POINTER(Model), C.POINTER(Config), C.c_int64,
                                      C.POINTER(C.c_int64), _d, _d, C.POINTER(C.c_int64),
                                      C.c_int32, _d, C.c_char_p, C.c_size_t]
        L.ref_solve_cells_ex.restype = C.c_int
        L.ref_solve_cells_ex.argtypes = [C.POINTER(Grid), _d, C.POINTER(Boundary),
                                         C.POINTER(Model), C.POINTER(Config), C.c_int64,
                                         C.POINTER(C.c_int64), _d, _d, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64), C.c_int32, _d, C.c_char_p,
                                         C.c_size_t]
        L.ref_trace_rays.restype = C.c_int
        L.ref_trace_rays.argtypes = [C.POINTER(Grid), _d, C.POINTER(Boundary),
                                     C.POINTER(Model), C.POINTER(Config), C.c_double,
                                     C.c_double, C.c_int64, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_uint32), _d, C.POINTER(RayResult),
                                     C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]
        L.ref_build_cdfs.restype = C.c_int
        L.ref_build_cdfs.argtypes = [C.POINTER(Model), C.c_double, _d, _d, C.c_char_p,
                                     C.c_size_t]
        L.ref_planck_mean.restype = C.c_int
        L.ref_planck_mean.argtypes = [C.POINTER(Model), C.c_double, _d, C.c_char_p,
                                      C.c_size_t]
        L.ref_interp.restype = C.c_int
        L.ref_interp.argtypes = [C.POINTER(Model), C.c_int, C.c_int, C.c_double, _d, _d,
                                 C.c_char_p, C.c_size_t]
        L.ref_uniform.restype = C.c_double
        L.ref_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]
        L.ref_build_hierarchy.restype = C.c_int
        L.ref_build_hierarchy.argtypes = [C.POINTER(Grid), _d, C.c_int, C.c_int,
                                          C.POINTER(Grid), _d, C.c_int64, C.c_char_p,
                                          C.c_size_t]
        _lib = L
    return _lib


class RefError(RuntimeError):
    pass


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def _check(rc, buf):
    if rc != 0:
        raise RefError(buf.value.decode(errors="replace"))


def solve(grid: Grid, temperature, boundary: Boundary, model, config: Config):
    """Reference ermc::solve. Returns (q_r, std_dev, steps, total, wall)."""
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    n = grid.nx * grid.ny * grid.nz
    q, sd = np.zeros(n), np.zeros(n)
    steps = np.zeros(config.n_levels, dtype=np.int64)
    sol = Solution(_p(q), _p(sd), _p(steps, C.c_int64), 0, 0.0)
    buf = C.create_string_buffer(2048)
    _check(lib().ref_solve(C.byref(grid), _p(t), C.byref(boundary), C.byref(model.desc),
                           C.byref(config), C.byref(sol), buf, len(buf)), buf)
    return q, sd, steps, int(sol.total_steps), float(sol.wall_time)


def solve_cells(grid, temperature, boundary, model, config, cells, threads=None):
    """Cell-subset replay through the reference's public init_ray/march API
    (bitwise solve() for those cells). Returns (q, sd, steps, wall)."""
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    q, sd = np.zeros(len(cells)), np.zeros(len(cells))
    steps = np.zeros(config.n_levels, dtype=np.int64)
    wall = C.c_double()
    nt = threads or os.cpu_count() or 1
    buf = C.create_string_buffer(2048)
    _check(lib().ref_solve_cells(C.byref(grid), _p(t), C.byref(boundary),
                                 C.byref(model.desc), C.byref(config), len(cells),
                                 _p(cells, C.c_int64), _p(q), _p(sd), _p(steps, C.c_int64),
                                 nt, C.byref(wall), buf, len(buf)), buf)
    return q, sd, steps, wall.value


def solve_cells_steps(grid, temperature, boundary, model, config, cells, threads=None):
    """solve_cells plus each selected cell's march steps (summed over its
    rays and levels). Returns (q, sd, steps_per_level, cell_steps, wall)."""
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    q, sd = np.zeros(len(cells)), np.zeros(len(cells))
    steps = np.zeros(config.n_levels, dtype=np.int64)
    cell_steps = np.zeros(len(cells), dtype=np.int64)
    wall = C.c_double()
    nt = threads or os.cpu_count() or 1
    buf = C.create_string_buffer(2048)
    _check(lib().ref_solve_cells_ex(C.byref(grid), _p(t), C.byref(boundary),
                                    C.byref(model.desc), C.byref(config), len(cells),
                                    _p(cells, C.c_int64), _p(q), _p(sd),
                                    _p(steps, C.c_int64), _p(cell_steps, C.c_int64), nt,
                                    C.byref(wall), buf, len(buf)), buf)
    return q, sd, steps, cell_steps, wall.value


def trace_rays(grid, temperature, boundary, model, config, t_max, qe, cells, rays,
               dirs=None):
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    rays = np.ascontiguousarray(rays, dtype=np.uint32)
    n = len(cells)
    out = (RayResult * n)()
    lvl = np.zeros(n * config.n_levels, dtype=np.int64)
    dptr = None
    if dirs is not None:
        dirs = np.ascontiguousarray(dirs, dtype=np.float64).ravel()
        dptr = _p(dirs)
    buf = C.create_string_buffer(2048)
    _check(lib().ref_trace_rays(C.byref(grid), _p(t), C.byref(boundary), C.byref(model.desc),
                                C.byref(config), t_max, qe, n, _p(cells, C.c_int64),
                                _p(rays, C.c_uint32), dptr, out, _p(lvl, C.c_int64), buf,
                                len(buf)), buf)
    return list(out), lvl.reshape(n, config.n_levels)


def build_cdfs(model, t_max):
    band = np.zeros(model.n_bands)
    quad = np.zeros(model.n_bands * model.n_quad)
    buf = C.create_string_buffer(2048)
    _check(lib().ref_build_cdfs(C.byref(model.desc), t_max, _p(band), _p(quad), buf,
                                len(buf)), buf)
    return band, quad.reshape(model.n_bands, model.n_quad)


def planck_mean(model, t):
    out = C.c_double()
    buf = C.create_string_buffer(2048)
    _check(lib().ref_planck_mean(C.byref(model.desc), t, C.byref(out), buf, len(buf)), buf)
    return out.value


def uniform(seed, cell, ray, draw):
    return lib().ref_uniform(seed, cell, ray, draw)


def hierarchy(grid, temperature, n_levels, ratio):
    t = np.ascontiguousarray(temperature, dtype=np.float64).ravel()
    grids = (Grid * n_levels)()
    cap = len(t) * 2 + 16
    out = np.zeros(cap)
    buf = C.create_string_buffer(2048)
    _check(lib().ref_build_hierarchy(C.byref(grid), _p(t), n_levels, ratio, grids, _p(out),
                                     cap, buf, len(buf)), buf)
    fields, off = [], 0
    for g in grids:
        n = g.nx * g.ny * g.nz
        fields.append(out[off:off + n].copy())
        off += n
    return list(grids), fields


# ---- the reference's own case library (via its pybind module) -------------

def ref_module():
    """The reference's `_ermc` pybind module built into oracle/_ref."""
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import _ermc  # noqa: PLC0415
    return _ermc


def read_ktab_arrays(path: str) -> capi.ModelArrays:
    """Plain numpy reader of a KTAB1 file (reference io.cpp:63-128)."""
    raw = Path(path).read_bytes()
    end = raw.index(b"\ndata\n") + len(b"\ndata\n")
    nb = nq = nt = 0
    temps, bands, quad = [], [], []
    for line in raw[:end].decode().splitlines()[1:]:
        f = line.split()
        if not f or f[0] == "data":
            continue
        if f[0] == "nbands":
            nb = int(f[1])
        elif f[0] == "nq":
            nq = int(f[1])
        elif f[0] == "ntemps":
            nt = int(f[1])
        elif f[0] == "temps":
            temps = [float(x) for x in f[1:]]
        elif f[0] == "band":
            bands.append([float(x) for x in f[1:4]])
        elif f[0] == "quad":
            quad.append([float(x) for x in f[1:3]])
    payload = np.frombuffer(raw[end:], dtype="<f8")
    k = payload[: nb * nq * nt].copy()
    ib = payload[nb * nq * nt: nb * nq * nt + nb * nt].copy()
    b = np.array(bands)
    qd = np.array(quad)
    return capi.ModelArrays(b[:, 0], b[:, 1], b[:, 2], qd[:, 0], qd[:, 1], temps, k, ib)


def read_tfld_arrays(path: str):
    raw = Path(path).read_bytes()
    end = raw.index(b"\ndata\n") + len(b"\ndata\n")
    hdr = {}
    for line in raw[:end].decode().splitlines()[1:]:
        f = line.split()
        if f and f[0] != "data":
            hdr[f[0]] = f[1:]
    dims = [int(x) for x in hdr["dims"]]
    sp = [float(x) for x in hdr["spacing"]]
    org = [float(x) for x in hdr.get("origin", ["0", "0", "0"])]
    vals = np.frombuffer(raw[end:], dtype="<f8")[: dims[0] * dims[1] * dims[2]].copy()
    return capi.make_grid(dims, sp, org), vals


def ref_case(name: str, grid_n: int = 0):
    """(grid, T, boundary, model_arrays, case) of the reference's make_case,
    exported through its own TFLD1/KTAB1 writers (bitwise inputs)."""
    R = ref_module()
    vc = R.make_case(name, grid_n)
    with tempfile.TemporaryDirectory() as td:
        R.write_tfld(os.path.join(td, "f.tfld"), vc.field)
        R.write_ktab(os.path.join(td, "m.ktab"), vc.model)
        grid, t = read_tfld_arrays(os.path.join(td, "f.tfld"))
        model = read_ktab_arrays(os.path.join(td, "m.ktab"))
    b = vc.boundary
    kind = [capi.PERIODIC if k == R.AxisKind.periodic else capi.WALL for k in b.kind]
    bnd = capi.make_boundary(kind, [(w.temperature, w.emissivity) for w in b.lo],
                             [(w.temperature, w.emissivity) for w in b.hi])
    return grid, t, bnd, model, vc
