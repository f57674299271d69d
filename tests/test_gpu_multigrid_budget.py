"""Multigrid step caps against max_steps, at the boundaries of the per-level
step budgets (trace_common.cuh set_level_budgets): the reference checks
max_steps before demotion (tracer.cpp:88-101), so a ray whose step count
reaches max_steps exactly where a level's cap ends stops there; one step more
and it demotes. Steps per level and Q_r against the reference's solve(), for
the black-wall multigrid tracer and the position-tracking one (grey walls).
"""
from __future__ import annotations

import numpy as np
import pytest

import refshim
from helpers import assert_fp64_parity
from paper_1810_00188_b200 import capi
from paper_1810_00188_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("walls", ["black", "grey"])
@pytest.mark.parametrize("levels,cap,max_steps", [
    (3, 5, 10),   # max_steps == the end of level 1's cap: stop, no demotion
    (3, 5, 11),   # one more: demote, one step on level 2
    (3, 5, 5),    # == level 0's cap: stop on level 0
    (4, 2, 7),    # inside level 3 (uncapped)
    (3, 0, 4),    # zero caps: straight to the coarsest level
])
def test_budget_edges_match_reference(walls, levels, cap, max_steps):
    g, t, b, m = W.channel_case(16, "nongrey16")[:4]
    if walls == "grey":
        b = capi.make_boundary((capi.PERIODIC, capi.WALL, capi.PERIODIC),
                               [(0.0, 1.0), (W.T_WALL_LO, 0.7), (0.0, 1.0)],
                               [(0.0, 1.0), (W.T_WALL_HI, 0.5), (0.0, 1.0)])
    cfg = capi.config_struct(rays_per_cell=8, seed=31, n_levels=levels,
                             steps_per_level=cap, max_steps=max_steps)
    try:
        rq, rsd, rsteps, rtotal, _ = refshim.solve(g, t, b, m, cfg)
    except refshim.RefError as exc:  # a config the reference rejects: so must we
        with pytest.raises(capi.ErmcError) as info:
            capi.solve(g, t, b, m, cfg)
        assert str(info.value) == str(exc)
        return
    q, sd, st, tot, _ = capi.solve(g, t, b, m, cfg)
    assert list(st) == list(rsteps)
    assert tot == rtotal
    assert_fp64_parity(q, rq, sd, rsd)
    assert max(np.nonzero(np.asarray(st))[0]) <= levels - 1
