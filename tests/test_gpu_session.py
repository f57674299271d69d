"""Sessions, chunking and error paths on the GPU, each against the reference
CPU solver (oracle/_ref) rather than against another GPU run.

* the asynchronous session (the DNS-coupling API):
  results of solve_async / wait and of a set_field on one stream followed by
  a solve on another stream match the reference; set_field while a solve is
  pending is refused;
* the multi-chunk path (per-ray buffer budget forced small with
  ERMC_QRAY_BUDGET): a cell range not starting at 0 split in many chunks
  matches the reference and the unchunked solve byte for byte;
* an error raised in a non-first chunk gives the reference's message
  (workers = 1: the first failing (cell, ray) in order);
* a table with a non-finite Ib next to a node the field sits on exactly:
  the reference's interp takes its frac == 0 shortcut and succeeds
  (spectral.cpp:179-205); so must the GPU.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import refshim
from helpers import assert_fp64_parity
from paper_1810_00188_b200 import capi
from paper_1810_00188_b200 import workloads as W
import paper_1810_00188_b200 as E

pytestmark = pytest.mark.gpu


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_async_session_and_cross_stream_set_field_match_reference():
    import torch
    g, t, b, m = W.channel_case(16, "nongrey16")[:4]
    n = g.nx * g.ny * g.nz
    cfg = capi.config_struct(rays_per_cell=32, seed=5)
    s = capi.Session(g, b, m, cfg)
    td = _dev(t)
    s.set_field(td.data_ptr(), True, 0)
    q = torch.empty(n, dtype=torch.float64, device="cuda")
    sd = torch.empty_like(q)
    s.solve_async(0, n, q.data_ptr(), sd.data_ptr(), 0)
    with pytest.raises(capi.ErmcError, match="pending"):
        s.set_field(td.data_ptr(), True, 0)
    st = s.wait()
    rq, rsd, rsteps, rtotal, _ = refshim.solve(g, t, b, m, cfg)
    assert list(st) == list(rsteps)
    assert_fp64_parity(q.cpu().numpy(), rq, sd.cpu().numpy(), rsd)

    # Next "DNS step": the new field is produced and handed over on stream A,
    # the solve is enqueued on stream B right away (no host sync between).
    t2 = t * 0.97 + 20.0
    a_st, b_st = torch.cuda.Stream(), torch.cuda.Stream()
    src = _dev(t2)
    torch.cuda.synchronize()
    with torch.cuda.stream(a_st):
        td2 = torch.empty_like(src)
        td2.copy_(src * 1.0)  # produced on A
    s.set_field(td2.data_ptr(), True, a_st.cuda_stream)
    q2 = torch.empty_like(q)
    sd2 = torch.empty_like(q)
    s.solve_async(0, n, q2.data_ptr(), sd2.data_ptr(), b_st.cuda_stream)
    st2 = s.wait()
    rq2, rsd2, rsteps2, _, _ = refshim.solve(g, t2, b, m, cfg)
    assert list(st2) == list(rsteps2)
    assert_fp64_parity(q2.cpu().numpy(), rq2, sd2.cpu().numpy(), rsd2)
    s.close()


@pytest.mark.parametrize("precision", [capi.FP64, capi.FP32])
def test_many_chunks_offset_range_matches_reference(precision, monkeypatch):
    g, t, b, m = W.channel_case(16, "nongrey16")[:4]
    lo, hi = 700, 3500
    cfg = capi.config_struct(rays_per_cell=16, seed=8, precision=precision)
    q0, sd0, st0, tot0, _ = capi.solve(g, t, b, m, cfg, cell_range=(lo, hi))
    # 256 cells x 16 rays x (8 B q_ray + 8 B sort keys) per chunk: 11 chunks
    monkeypatch.setenv("ERMC_QRAY_BUDGET", str(256 * 16 * 16))
    q, sd, st, tot, _ = capi.solve(g, t, b, m, cfg, cell_range=(lo, hi))
    assert np.array_equal(q, q0) and np.array_equal(sd, sd0) and tot == tot0
    if precision == capi.FP64:
        cfg64 = capi.config_struct(rays_per_cell=16, seed=8)
        rq, rsd, rsteps, _ = refshim.solve_cells(g, t, b, m, cfg64, np.arange(lo, hi))
        assert tot == int(rsteps.sum())
        assert_fp64_parity(q, rq, sd, rsd)


def _grey_slab_with_bad_ib(node_t):
    """Grey 24x8x8 slab, kappa 50 (rays die within ~5 cells), Ib of every
    band set to +inf at the temperature node `node_t`."""
    grid = capi.make_grid((24, 8, 8), (1.0 / 24, 1.0 / 8, 1.0 / 8))
    model = E.grey_model(50.0, E.make_planck_bands(900.0, 1100.0, 8),
                         E.make_temp_grid(900.0, 1100.0, 10.0))
    ma = capi.model_from_ermc(model)
    ib = ma.ib_table.reshape(ma.n_bands, -1).copy()
    ib[:, int(round((node_t - 900.0) / 10.0))] = np.inf
    ma = capi.ModelArrays(ma.nu_lo, ma.nu_hi, ma.nu_center, ma.g_points, ma.g_weights,
                          ma.temps, ma.k_table, ib)
    b = capi.make_boundary((capi.WALL, capi.PERIODIC, capi.PERIODIC),
                           [(950.0, 1.0), (0.0, 1.0), (0.0, 1.0)],
                           [(950.0, 1.0), (0.0, 1.0), (0.0, 1.0)])
    return grid, ma, b


def test_error_in_a_later_chunk_has_the_reference_message(monkeypatch):
    # Ib(930 K) = inf: only rays that enter the 925 K planes x >= 20
    # fail; those start at x >= 15, i.e. in the last chunks.
    grid, m, b = _grey_slab_with_bad_ib(930.0)
    t = np.full(24 * 64, 950.0)
    t[20 * 64:] = 925.0
    cfg = capi.config_struct(rays_per_cell=8, seed=3, workers=1)
    with pytest.raises(refshim.RefError) as ref_err:
        refshim.solve(grid, t, b, m, cfg)
    assert "non-finite" in str(ref_err.value)
    cell = int(str(ref_err.value).split("cell ")[1].split()[0])
    assert cell >= 14 * 64
    for budget in (None, str(2 * 64 * 8 * 16)):  # one chunk; 2 x-planes per chunk
        if budget:
            monkeypatch.setenv("ERMC_QRAY_BUDGET", budget)
        with pytest.raises(capi.ErmcError) as gpu_err:
            capi.solve(grid, t, b, m, cfg)
        assert str(gpu_err.value) == str(ref_err.value)


@pytest.mark.parametrize("precision", [capi.FP64, capi.FP32])
def test_nonfinite_ib_beside_an_exact_node_succeeds_like_the_reference(precision):
    # Ib(1010 K) = inf; every cell sits exactly on the 1000 K or
    # 950 K node, T_max = 1000 K: interp returns the node value (frac == 0)
    # and never touches the inf — the reference solves without error.
    grid, m, b = _grey_slab_with_bad_ib(1010.0)
    t = np.full(24 * 64, 950.0)
    t[::3] = 1000.0
    cfg = capi.config_struct(rays_per_cell=16, seed=4, precision=precision)
    rq, rsd, rsteps, rtotal, _ = refshim.solve(grid, t, b, m, capi.config_struct(rays_per_cell=16,
                                                                                 seed=4))
    if precision == capi.FP32:  # normalised fp32 records cannot hold it: refused
        with pytest.raises(capi.ErmcError, match="finite k / Ib tables"):
            capi.solve(grid, t, b, m, cfg)
        return
    q, sd, st, tot, _ = capi.solve(grid, t, b, m, cfg)
    assert tot == rtotal
    assert_fp64_parity(q, rq, sd, rsd)
