"""Host-side setup of the product (table builders, CDFs, Planck mean, file
formats, validation) against the reference — no GPU needed. The trace
kernel consumes these arrays, so they must be bitwise the reference's.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1810_00188_b200 as E
import refshim
from helpers import GOLDEN, load_model
from paper_1810_00188_b200 import capi
from paper_1810_00188_b200 import workloads as W

needs_ref = pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")


def _models(mod):
    sp = mod.elsasser_spectrum(mod.make_temp_grid(450.0, 1050.0, 5.0))
    small = mod.elsasser_spectrum(mod.make_temp_grid(500.0, 1500.0, 250.0)) \
        if mod is not E else E.elsasser_spectrum(E.make_temp_grid(500.0, 1500.0, 250.0))
    return [
        mod.grey_model(1.0, mod.make_planck_bands(900.0, 1100.0, 64),
                       mod.make_temp_grid(900.0, 1100.0, 10.0)),
        mod.grey_model(2.0, mod.make_planck_bands(450.0, 1550.0, 8),
                       mod.make_temp_grid(450.0, 1550.0, 25.0),
                       mod.QuadratureSet.gauss_legendre(4)),
        mod.grey_model(0.5, mod.make_planck_bands(2.0, 90.0, 64),
                       mod.make_temp_grid(2.0, 90.0, 0.25)),
        mod.build_k_distribution(sp, mod.make_bands(sp.nu_grid[0], sp.nu_grid[-1] + 1e-6, 16),
                                 mod.QuadratureSet.gauss_legendre(16)),
        mod.build_k_distribution(small, mod.make_bands(small.nu_grid[0],
                                                       small.nu_grid[-1] + 1e-6, 119),
                                 mod.QuadratureSet.gauss_legendre(8)),
    ]


@needs_ref
def test_builders_write_identical_ktab_bytes(tmp_path):
    R = refshim.ref_module()
    for i, (a, b) in enumerate(zip(_models(R), _models(E))):
        pa, pb = tmp_path / f"r{i}.ktab", tmp_path / f"m{i}.ktab"
        R.write_ktab(str(pa), a)
        E.write_ktab(str(pb), b)
        assert pa.read_bytes() == pb.read_bytes(), i
        for t in (500.0, 777.7, 1000.0):
            try:
                assert a.planck_mean(t) == b.planck_mean(t)
            except RuntimeError:
                with pytest.raises(RuntimeError):
                    b.planck_mean(t)


@needs_ref
def test_gauss_legendre_bitwise():
    R = refshim.ref_module()
    for n in (1, 2, 3, 4, 8, 16, 32, 96):
        a, b = R.QuadratureSet.gauss_legendre(n), E.QuadratureSet.gauss_legendre(n)
        assert a.g_points == b.g_points and a.weights == b.weights


def test_cabi_cdfs_and_planck_mean_match_golden():
    z = np.load(GOLDEN / "cdfs_channel16.npz")
    m = load_model(z)
    for tm in (573.0, 800.0, 955.0):
        bc, qc = capi.build_cdfs(m, tm)
        assert np.array_equal(bc, z[f"band_{tm:g}"]) and np.array_equal(qc, z[f"quad_{tm:g}"])
        assert capi.planck_mean(m, tm) == z[f"kp_{tm:g}"][0]


def test_cpp_api_cdfs_match_cabi():
    m = W.nongrey_channel_model(16)
    bc, qc = E.build_cdfs(m, 955.0)
    b2, q2 = capi.build_cdfs(capi.model_from_ermc(m), 955.0)
    assert np.array_equal(np.array(bc), b2) and np.array_equal(np.array(qc), q2)


@needs_ref
def test_interpolation_matches_reference():
    R = refshim.ref_module()
    a, b = _models(R)[3], _models(E)[3]
    rng = np.random.default_rng(0)
    for t in np.concatenate([rng.uniform(450.0, 1050.0, 200), [450.0, 1050.0, 455.0, 1045.0]]):
        for n in (0, 7, 15):
            for g in (0, 9, 15):
                assert a.interp_k(n, g, t) == b.interp_k(n, g, t)
            assert a.interp_ib(n, t) == b.interp_ib(n, t)


def test_interpolation_errors_outside_table():
    m = E.grey_model(1.0, E.make_planck_bands(500.0, 1500.0, 16),
                     E.make_temp_grid(500.0, 1500.0, 100.0))
    with pytest.raises(RuntimeError, match="outside table range"):
        m.interp_k(0, 0, 499.9)
    with pytest.raises(RuntimeError):
        m.planck_mean(1501.0)


def test_table_validation_messages():
    bands = E.make_bands(100.0, 200.0, 2)
    q = E.QuadratureSet.single_point()
    with pytest.raises(RuntimeError, match="k_table entries must be non-negative"):
        E.SpectralModel(bands, q, [500.0, 600.0], [1.0, -1.0, 1.0, 1.0], [1.0] * 4)
    with pytest.raises(RuntimeError, match="temperature grid must be ascending"):
        E.SpectralModel(bands, q, [600.0, 500.0], [1.0] * 4, [1.0] * 4)
    with pytest.raises(RuntimeError, match="grey_model: kappa must be non-negative"):
        E.grey_model(-1.0, bands, [500.0, 600.0])
    with pytest.raises(RuntimeError, match="make_planck_bands: need at least 8 bands"):
        E.make_planck_bands(500.0, 600.0, 4)


@needs_ref
def test_file_formats_byte_compatible(tmp_path):
    R = refshim.ref_module()
    for mod, tag in ((R, "r"), (E, "m")):
        f = mod.TemperatureField()
        g = mod.CartesianGrid()
        g.nx, g.ny, g.nz = 3, 4, 5
        g.dx, g.dy, g.dz = 0.125, 0.3, 1.0 / 7
        g.origin = [0.25, -1.0, 3.5]
        f.grid = g
        f.values = [300.0 + 1.0 / (c + 1) for c in range(60)]
        mod.write_tfld(str(tmp_path / f"{tag}.tfld"), f)
    assert (tmp_path / "r.tfld").read_bytes() == (tmp_path / "m.tfld").read_bytes()
    back = E.read_tfld(str(tmp_path / "r.tfld"))
    assert back.grid.dz == 1.0 / 7 and back.values[5] == 300.0 + 1.0 / 6
    assert E.file_hash(str(tmp_path / "r.tfld")) == R.file_hash(str(tmp_path / "r.tfld"))
    km = _models(E)[1]
    E.write_ktab(str(tmp_path / "m.ktab"), km)
    back = R.read_ktab(str(tmp_path / "m.ktab"))
    assert back.planck_mean(1000.0) == km.planck_mean(1000.0)


def test_read_errors(tmp_path):
    p = tmp_path / "bad.tfld"
    p.write_bytes(b"TFLD2\n")
    with pytest.raises(RuntimeError, match="bad magic"):
        E.read_tfld(str(p))
    p.write_bytes(b"TFLD1\ndims 2 2 2\nspacing 1 1 1\ndata\n" + b"\0" * 16)
    with pytest.raises(RuntimeError, match="truncated binary payload"):
        E.read_tfld(str(p))


def test_solve_config_validation_is_host_side():
    g = E.CartesianGrid()
    f = E.TemperatureField()
    f.grid = g
    f.values = [1000.0]
    m = E.grey_model(1.0, E.make_planck_bands(900.0, 1100.0, 8), E.make_temp_grid(900.0, 1100.0, 50.0))
    b = E.BoundarySpec()
    cfg = E.SolveConfig()
    cfg.rays_per_cell = 0
    with pytest.raises(RuntimeError, match="rays_per_cell must be >= 1"):
        E.solve(g, f, b, m, cfg)
    cfg = E.SolveConfig()
    cfg.tolerance = 1.5
    with pytest.raises(RuntimeError, match=r"tolerance must be in \(0,1\)"):
        E.solve(g, f, b, m, cfg)
    bad = E.TemperatureField()
    bad.grid = g
    bad.values = [1000.0, 1000.0]
    with pytest.raises(RuntimeError, match="value count does not match grid"):
        E.solve(g, bad, b, m, E.SolveConfig())


def test_solve_without_gpu_fails_loudly():
    # There is no CPU fallback: without a device the solve reports it.
    if capi.load().ermc_b200_device_count() > 0:
        pytest.skip("a GPU is present")
    g, t, b, m, _ = W.channel_case(4, "grey")
    with pytest.raises(capi.ErmcError, match="no CUDA device"):
        capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=2))
    with pytest.raises(capi.ErmcError, match="no CUDA device"):
        capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=2, n_devices=4))


def test_n_devices_validation():
    g, t, b, m, _ = W.channel_case(4, "grey")
    with pytest.raises(capi.ErmcError, match="n_devices must be >= 0"):
        capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=2, n_devices=-1))
    c = E.SolveConfig()
    assert c.n_devices == 1


def test_channel_field_matches_survey_range():
    t = W.channel_field(64)
    assert 575.0 < t.min() < 577.0 and 951.0 < t.max() < 953.0  # [576, 952]


@needs_ref
def test_lbl_model_matches_reference_tables():
    # lbl_model (reference oracles.cpp:232-264), restated on the reference's
    # own spectrum and planck_intensity: one band per sample, midpoint edges,
    # kappa transposed to [sample][T], Ib(nu_s, T) (0 at T <= 0).
    R = refshim.ref_module()
    for temps in ([500.0, 1000.0, 1500.0], [450.0 + 50.0 * j for j in range(13)]):
        sp = R.elsasser_spectrum(temps)
        nu = np.asarray(sp.nu_grid)
        kap = np.asarray(sp.kappa)
        m = E.lbl_model(E.elsasser_spectrum(temps))
        assert m.n_bands() == len(nu) and m.n_quad() == 1
        assert np.array_equal(np.asarray(m.k_table()), kap.T.reshape(-1))
        ib = np.array([[R.planck_intensity(v, t) if t > 0 else 0.0 for t in temps]
                       for v in nu])
        assert np.array_equal(np.asarray(m.ib_table()), ib.reshape(-1))
        lo = np.array([b.nu_lo for b in m.bands()])
        hi = np.array([b.nu_hi for b in m.bands()])
        assert lo[0] == nu[0] - 0.5 * (nu[1] - nu[0])
        assert hi[-1] == nu[-1] + 0.5 * (nu[-1] - nu[-2])
        assert np.array_equal(lo[1:], 0.5 * (nu[:-1] + nu[1:]))
        assert np.array_equal(hi[:-1], 0.5 * (nu[:-1] + nu[1:]))


def test_lbl_flat_spectrum_is_the_grey_model_bitwise():
    # test_oracles.cpp:124-137
    temps = [500.0, 1000.0, 1500.0]
    grey = E.LineSpectrum()
    grey.temps = temps
    grey.nu_grid = [400.0 + 2.5 * i for i in range(201)]
    grey.kappa = [[2.0] * 201 for _ in temps]
    lbl = E.lbl_model(grey)
    direct = E.grey_model(2.0, lbl.bands(), temps, E.QuadratureSet.single_point())
    assert lbl.k_table() == direct.k_table()
    assert lbl.ib_table() == direct.ib_table()
    assert lbl.n_bands() == 201 and lbl.n_quad() == 1


def test_lbl_memory_cap_is_enforced():
    # test_oracles.cpp:158-162: the cap is checked before any table is built.
    sp = E.elsasser_spectrum([500.0, 1000.0, 1500.0])
    with pytest.raises(RuntimeError, match="bytes"):
        E.lbl_model(sp, 1024)
    grid = E.CartesianGrid()
    field = E.TemperatureField()
    with pytest.raises(RuntimeError, match="lbl_model: tables would need"):
        E.lbl_reference(grid, field, E.BoundarySpec(), sp, E.SolveConfig(), 1024)
