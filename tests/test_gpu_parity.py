"""GPU parity: the sm_100a trace kernel vs the reference CPU solver.

Every test drives the product through the C-ABI (paper_1810_00188_b200.capi)
and the checker through oracle/refshim (the unmodified reference compiled
into oracle/_ref). Case definitions come from the reference's own
make_case (proj/src/cases.cpp:211-295) exported through its KTAB1/TFLD1
writers, so both sides consume identical bytes.
"""
from __future__ import annotations

import numpy as np
import pytest

import refshim
from helpers import allowed_3sigma, assert_fp64_parity, three_sigma_violations
from paper_1810_00188_b200 import capi
from paper_1810_00188_b200 import workloads as W

pytestmark = pytest.mark.gpu

# (case, grid_n, rays, seed) — the reference's verification library at sizes
# the CPU reference finishes in seconds.
CASES = [
    ("isothermal", 8, 64, 1),
    ("grey-lin1", 10, 64, 11),
    ("grey-parab", 12, 64, 3),
    ("box-sin-05", 8, 32, 4),
    ("box-sin-5", 10, 32, 2),
    ("epsw-11", 8, 32, 6),
    ("epsw-01", 8, 32, 8),
    ("epsw-low", 8, 24, 5),
    ("nb-parab", 10, 64, 7),
    ("nb-3dimens", 8, 32, 9),
]


def _solve_both(grid, t, b, m, cfg):
    g = capi.solve(grid, t, b, m, cfg)
    r = refshim.solve(grid, t, b, m, cfg)
    return g, r


@pytest.mark.parametrize("name,n,rays,seed", CASES)
def test_fp64_matches_reference(name, n, rays, seed):
    grid, t, b, m, _ = refshim.ref_case(name, n)
    cfg = capi.config_struct(rays_per_cell=rays, seed=seed)
    (q, sd, steps, total, _), (rq, rsd, rsteps, rtotal, _) = _solve_both(grid, t, b, m, cfg)
    assert total == rtotal
    assert list(steps) == list(rsteps)
    rep = assert_fp64_parity(q, rq, sd, rsd)
    print(name, rep)


def test_isothermal_is_bitwise_zero():
    # P1 (acceptance.cpp:57-74) at the reference's default 16^3, R = 500.
    grid, t, b, m, _ = refshim.ref_case("isothermal", 0)
    cfg = capi.config_struct(rays_per_cell=500)
    q, sd, _, total, _ = capi.solve(grid, t, b, m, cfg)
    assert np.all(q == 0.0) and np.all(sd == 0.0)
    assert total > 0


@pytest.mark.parametrize("variant", [
    dict(specular_walls=1),
    dict(volume_sampling=1),
    dict(tolerance=1e-6),
    dict(max_steps=7),
    dict(n_levels=3, steps_per_level=4),
    dict(n_levels=2, steps_per_level=3, coarsen_ratio=3),
    dict(sorting=1),
])
def test_fp64_option_variants(variant):
    grid, t, b, m, _ = refshim.ref_case("epsw-low", 8)
    cfg = capi.config_struct(rays_per_cell=32, seed=21, **variant)
    (q, sd, steps, total, _), (rq, rsd, rsteps, rtotal, _) = _solve_both(grid, t, b, m, cfg)
    assert total == rtotal, variant
    assert list(steps) == list(rsteps), variant
    assert_fp64_parity(q, rq, sd, rsd)


def test_fp64_multigrid_3d_walls():
    grid, t, b, m, _ = refshim.ref_case("nb-3dimens", 12)
    cfg = capi.config_struct(rays_per_cell=32, seed=4, n_levels=4, steps_per_level=2)
    (q, sd, steps, total, _), (rq, rsd, rsteps, rtotal, _) = _solve_both(grid, t, b, m, cfg)
    assert list(steps) == list(rsteps)
    assert_fp64_parity(q, rq, sd, rsd)


def test_fp64_channel_nongrey_matches_reference():
    # Config 3/4 geometry and tables at a CPU-sized grid.
    grid, t, b, m, _ = W.channel_case(16, "nongrey16")
    cfg = capi.config_struct(rays_per_cell=32, seed=2024)
    (q, sd, steps, total, _), (rq, rsd, rsteps, rtotal, _) = _solve_both(grid, t, b, m, cfg)
    assert total == rtotal
    assert_fp64_parity(q, rq, sd, rsd)


def test_fp64_channel_grey_tau_sweep():
    for tau in (0.1, 1.0, 10.0):
        grid, t, b, m, _ = W.channel_case(12, "grey", tau=tau)
        cfg = capi.config_struct(rays_per_cell=16, seed=5)
        (q, sd, steps, total, _), (rq, rsd, rsteps, rtotal, _) = _solve_both(grid, t, b, m, cfg)
        assert total == rtotal, tau
        assert_fp64_parity(q, rq, sd, rsd)


def test_slab_ranges_reassemble_bitwise():
    # Multi-GPU sharding contract: x-slabs solved separately concatenate to
    # the full solve byte for byte (GPU analogue of P8).
    grid, t, b, m, _ = refshim.ref_case("nb-parab", 8)
    cfg = capi.config_struct(rays_per_cell=32, seed=13)
    q, sd, steps, total, _ = capi.solve(grid, t, b, m, cfg)
    n = grid.nx * grid.ny * grid.nz
    cuts = [0, 37, 64 * 3, n - 5, n]
    qs, sds, tot = [], [], 0
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        a, s_, st, tt, _ = capi.solve(grid, t, b, m, cfg, cell_range=(lo, hi))
        qs.append(a)
        sds.append(s_)
        tot += tt
    assert np.array_equal(np.concatenate(qs), q)
    assert np.array_equal(np.concatenate(sds), sd)
    assert tot == total


def test_repeat_is_deterministic():
    grid, t, b, m, _ = refshim.ref_case("grey-parab", 8)
    cfg = capi.config_struct(rays_per_cell=48, seed=99)
    a = capi.solve(grid, t, b, m, cfg)
    c = capi.solve(grid, t, b, m, cfg)
    assert np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1]) and a[3] == c[3]


def test_fp32_statistical_parity():
    grid, t, b, m, _ = W.channel_case(16, "nongrey16")
    cfg64 = capi.config_struct(rays_per_cell=64, seed=31)
    cfg32 = capi.config_struct(rays_per_cell=64, seed=32, precision=capi.FP32)
    q64, sd64, _, t64, _ = capi.solve(grid, t, b, m, cfg64)
    q32, sd32, _, t32, _ = capi.solve(grid, t, b, m, cfg32)
    n = len(q64)
    bad = three_sigma_violations(q64, q32, sd64, sd32)
    assert bad <= allowed_3sigma(n), (bad, n)
    # Same seed: the fp32 kernel traces the reference's rays.
    cfg32s = capi.config_struct(rays_per_cell=64, seed=31, precision=capi.FP32)
    q32s, sd32s, _, t32s, _ = capi.solve(grid, t, b, m, cfg32s)
    assert abs(t32s - t64) <= 1e-3 * t64
    rel = np.abs(q32s - q64) / (np.abs(q64) + 1e-3 * np.max(np.abs(q64)))
    assert np.median(rel) < 1e-3, np.median(rel)


def test_device_rng_is_the_reference_stream():
    rng = np.random.default_rng(5)
    n = 20000
    cells = rng.integers(0, 2**40, n, dtype=np.uint64)
    rays = rng.integers(0, 2**31, n, dtype=np.uint32)
    draws = rng.integers(0, 64, n, dtype=np.uint32)
    for seed in (0, 17, 2**63 + 5):
        got = capi.uniform_device(seed, cells, rays, draws)
        want = np.array([refshim.uniform(seed, int(c), int(r), int(d))
                         for c, r, d in zip(cells, rays, draws)])
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name,n,variant", [
    ("epsw-low", 10, {}),                       # even grid: micro-brick tracer, grey walls
    ("epsw-low", 9, {}),                        # odd grid: linear-layout lean tracer
    ("nb-3dimens", 10, dict(specular_walls=1)),  # all walls, specular
    ("box-sin-5", 9, {}),
    ("nb-parab", 12, dict(volume_sampling=1)),
    ("nb-3dimens", 12, dict(n_levels=3, steps_per_level=3)),  # lean multigrid tracers
    ("epsw-low", 10, dict(n_levels=2, steps_per_level=4)),
])
def test_fp32_tracks_fp64_on_the_same_rays(name, n, variant):
    # Same seed: the fp32 kernel traces the reference's rays (same draws,
    # same (band, g)); per-cell results agree far inside the MC noise and the
    # step counts agree to 1e-3 (fp32 DDA ties resolve differently rarely).
    grid, t, b, m, _ = refshim.ref_case(name, n)
    q64, sd64, _, t64, _ = capi.solve(grid, t, b, m, capi.config_struct(
        rays_per_cell=32, seed=77, **variant))
    q32, sd32, _, t32, _ = capi.solve(grid, t, b, m, capi.config_struct(
        rays_per_cell=32, seed=77, precision=capi.FP32, **variant))
    assert abs(t32 - t64) <= 1e-3 * t64, (t32, t64)
    bad = three_sigma_violations(q64, q32, 0.1 * sd64, 0.1 * sd32)
    assert bad <= allowed_3sigma(len(q64)), bad


def _lbl_inputs(mod, n, t_fn, wall):
    g = mod.CartesianGrid()
    g.nx = g.ny = g.nz = n
    g.dx = g.dy = g.dz = 1.0 / n
    f = mod.TemperatureField()
    f.grid = g
    f.values = [t_fn((i + 0.5) / n) for i in range(n) for _ in range(n * n)]
    b = mod.BoundarySpec()
    b.lo = [mod.Wall(wall, 1.0)] * 3
    b.hi = [mod.Wall(wall, 1.0)] * 3
    return g, f, b


@pytest.mark.parametrize("profile", ["isothermal", "parab"])
def test_lbl_reference_matches_reference(profile):
    # lbl_reference (oracles.cpp:266-274) through the drop-in Python module:
    # the default Elsasser spectrum (8001 line-by-line bands, one g point)
    # on the test_oracles.cpp:117-163 temperature nodes.
    import paper_1810_00188_b200 as E
    R = refshim.ref_module()
    temps = [500.0, 1000.0, 1500.0]
    t_fn = (lambda x: 1000.0) if profile == "isothermal" else \
        (lambda x: 600.0 + 1600.0 * x * (1.0 - x))
    out = []
    for mod in (E, R):
        sp = mod.elsasser_spectrum(temps)
        assert len(sp.nu_grid) == 8001
        g, f, b = _lbl_inputs(mod, 6, t_fn, 1000.0 if profile == "isothermal" else 600.0)
        cfg = mod.SolveConfig()
        cfg.rays_per_cell = 40
        cfg.seed = 5
        out.append(mod.lbl_reference(g, f, b, sp, cfg))
    s, r = out
    if profile == "isothermal":
        assert all(q == 0.0 for q in s.q_r)
    assert s.total_steps == r.total_steps
    assert_fp64_parity(np.asarray(s.q_r), np.asarray(r.q_r),
                       np.asarray(s.std_dev), np.asarray(r.std_dev))


@pytest.mark.parametrize("n_devices", [2, 3])
def test_multi_device_split_is_byte_identical(n_devices):
    # ermc_config_t.n_devices: the range is split into contiguous parts on
    # (device + p) mod visible devices, one host thread each. On a one-GPU box
    # the parts share the device; the assembly and the result must not change.
    g, t, b, m = W.channel_case(24, "nongrey16")[:4]
    one = capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=32, seed=4))
    many = capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=32, seed=4,
                                                     n_devices=n_devices))
    assert np.array_equal(one[0], many[0]) and np.array_equal(one[1], many[1])
    assert list(one[2]) == list(many[2]) and one[3] == many[3]
    lo, hi = 1000, 9000
    part = capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=32, seed=4,
                                                     n_devices=n_devices), cell_range=(lo, hi))
    assert np.array_equal(part[0], one[0][lo:hi])


def test_edge_sizes_match_reference():
    # Degenerate inputs the reference accepts: one ray per cell (std_dev = 0,
    # solver.cpp:150-153), a one-cell grid, a one-cell-thick slab, an empty
    # cell range, and a max_steps cap that truncates most rays.
    grid, t, b, m, _ = refshim.ref_case("nb-parab", 6)
    for cfg in (capi.config_struct(rays_per_cell=1, seed=21),
                capi.config_struct(rays_per_cell=16, seed=22, max_steps=3)):
        (q, sd, steps, total, _), (rq, rsd, rsteps, rtotal, _) = _solve_both(grid, t, b, m, cfg)
        assert total == rtotal and list(steps) == list(rsteps)
        assert_fp64_parity(q, rq, sd, rsd)
        if cfg.rays_per_cell == 1:
            assert np.all(sd == 0.0)
    q, sd, steps, total, _ = capi.solve(grid, t, b, m, capi.config_struct(rays_per_cell=8),
                                        cell_range=(5, 5))
    assert q.size == 0 and total == 0
    for shape in ((1, 1, 1), (1, 5, 7), (9, 1, 1)):
        g = capi.make_grid(shape, (0.1, 0.2, 0.3))
        n = shape[0] * shape[1] * shape[2]
        tt = np.linspace(600.0, 1000.0, n) if n > 1 else np.array([900.0])
        bb = capi.make_boundary((capi.WALL, capi.PERIODIC, capi.WALL),
                                [(500.0, 1.0), (0.0, 1.0), (800.0, 0.3)],
                                [(1000.0, 0.5), (0.0, 1.0), (0.0, 1.0)])
        cfg = capi.config_struct(rays_per_cell=40, seed=23)
        (q, sd, steps, total, _), (rq, rsd, rsteps, rtotal, _) = _solve_both(g, tt, bb, m, cfg)
        assert total == rtotal, shape
        assert_fp64_parity(q, rq, sd, rsd)


def _solve_in_subprocess(env_extra, name, n, rays, seed, precision):
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = (
        "import sys, json, numpy as np\n"
        f"sys.path[:0] = [{str(root)!r}, {str(root / 'oracle')!r}]\n"
        "import refshim\n"
        "from paper_1810_00188_b200 import capi\n"
        f"g, t, b, m, _ = refshim.ref_case({name!r}, {n})\n"
        f"q, sd, st, tot, _ = capi.solve(g, t, b, m, capi.config_struct(rays_per_cell={rays}, "
        f"seed={seed}, precision={precision}))\n"
        "print(json.dumps([q.tobytes().hex(), sd.tobytes().hex(), int(tot)]))\n")
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         check=True).stdout.strip().splitlines()[-1]
    return json.loads(out)


@pytest.mark.parametrize("precision", [capi.FP64, capi.FP32])
def test_dispatch_order_never_changes_results(precision):
    # The narrow-band sorted dispatch (dispatch.cu) and its direction bins only
    # reorder the marching: byte-identical Q_r / sigma / steps with the sort
    # off, on, and on with 1 or 32 direction bins (P5 for the GPU schedule).
    runs = [_solve_in_subprocess(env, "nb-parab", 10, 48, 31, precision)
            for env in ({"ERMC_SORT": "0"}, {"ERMC_SORT": "1", "ERMC_SORT_DIRS": "1"},
                        {"ERMC_SORT": "1", "ERMC_SORT_DIRS": "32"},
                        {"ERMC_SORT": "1", "ERMC_SORT_TILE": "1000"},
                        {"ERMC_SORT": "1", "ERMC_SORT_BLOCK": "8"},  # cubic tiles, clipped
                        {"ERMC_SORT": "1", "ERMC_SORT_BLOCK": "4"})]
    assert all(r == runs[0] for r in runs[1:])


def test_async_session_overlaps_the_host_and_matches_sync():
    # session_solve_async returns while the solve runs (the host can advance a
    # DNS step meanwhile); wait() then gives the same bytes and
    # step counts as the synchronous call, and errors surface at wait().
    import time
    import torch
    g, t, b, m = W.channel_case(64, "nongrey16")[:4]
    n = g.nx * g.ny * g.nz
    cfg = capi.config_struct(rays_per_cell=32, seed=5)
    s = capi.Session(g, b, m, cfg)
    td = torch.from_numpy(t).cuda()
    s.set_field(td.data_ptr(), True, 0)
    q1 = torch.empty(n, dtype=torch.float64, device="cuda")
    sd1 = torch.empty_like(q1)
    st1 = s.solve(0, n, q1.data_ptr(), sd1.data_ptr(), 0)
    t_sync = s.timings()[0][2]
    q2 = torch.empty_like(q1)
    sd2 = torch.empty_like(q1)
    t0 = time.perf_counter()
    s.solve_async(0, n, q2.data_ptr(), sd2.data_ptr(), 0)
    enqueue_ms = (time.perf_counter() - t0) * 1e3
    with pytest.raises(capi.ErmcError, match="pending"):
        s.solve_async(0, n, q2.data_ptr(), sd2.data_ptr(), 0)
    st2 = s.wait()
    with pytest.raises(capi.ErmcError, match="no solve pending"):
        s.wait()
    assert torch.equal(q1, q2) and torch.equal(sd1, sd2) and list(st1) == list(st2)
    assert enqueue_ms < 0.5 * t_sync, (enqueue_ms, t_sync)
    s.close()


def test_fp32_brick_layouts_give_identical_bytes():
    # The fp32 field layout (2^3 or 4^3 micro-bricks) changes addressing only:
    # the same rays, the same arithmetic, byte-identical Q_r / sigma / steps.
    def run(env):
        import json
        import os
        import subprocess
        import sys
        from pathlib import Path
        root = Path(__file__).resolve().parent.parent
        code = (
            "import sys, json\n"
            f"sys.path[:0] = [{str(root)!r}]\n"
            "from paper_1810_00188_b200 import capi, workloads as W\n"
            "g, t, b, m = W.channel_case(32, 'nongrey16')[:4]\n"
            "q, sd, st, tot, _ = capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=16, "
            "seed=3, precision=capi.FP32))\n"
            "print(json.dumps([q.tobytes().hex(), sd.tobytes().hex(), int(tot)]))\n")
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                             capture_output=True, text=True, check=True).stdout
        return json.loads(out.strip().splitlines()[-1])
    assert run({"ERMC_BRICK": "1"}) == run({"ERMC_BRICK": "4"})
