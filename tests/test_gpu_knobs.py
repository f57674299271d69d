"""Scheduling knobs never change a result: the narrow-band sort's tile shape
(linear tiles `ERMC_SORT_BLOCK=0`, the default cubic tiles — the largest cube
with edge^3 R <= 2^16, clipped at the grid's faces — and a small ragged
edge) and the march windows (the default windows are compiled into the bench
kernels; any other value launches the runtime-bound kernels) give
byte-identical Q_r, sigma and step counts, single level in fp64 and fp32 and
3-level multigrid, on a grid no tile edge divides. The knobs are read once
per process, so each setting runs in its own.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = """
import sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_1810_00188_b200 import capi, workloads as W
g, t, b, m = W.channel_case(22, "nongrey16")[:4]
out = []
for prec, levels in ((capi.FP64, 1), (capi.FP32, 1), (capi.FP64, 3)):
    q, sd, st, tot, _ = capi.solve(g, t, b, m, capi.config_struct(
        rays_per_cell=24, seed=9, precision=prec, n_levels=levels, steps_per_level=3))
    out += [q, sd, np.asarray(st, dtype=np.float64)]
np.save({path!r}, np.concatenate(out))
"""

KNOBS = ["ERMC_SORT_BLOCK", "ERMC_INNER_STEPS", "ERMC_INNER_STEPS32", "ERMC_INNER_STEPS_MG"]


def _run(tmp_path, tag, **env_set):
    path = str(tmp_path / f"knobs_{tag}.npy")
    env = {k: v for k, v in os.environ.items() if k not in KNOBS}
    env.update({k: str(v) for k, v in env_set.items()})
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), path=path)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


def test_scheduling_knobs_never_change_results(tmp_path):
    default = _run(tmp_path, "default")  # cubic tiles, edge 13 at R = 24 (22 = 13 + 9)
    variants = {
        "linear": dict(ERMC_SORT_BLOCK=0),
        "ragged5": dict(ERMC_SORT_BLOCK=5),
        "windows": dict(ERMC_INNER_STEPS=24, ERMC_INNER_STEPS32=40, ERMC_INNER_STEPS_MG=40),
    }
    for tag, env_set in variants.items():
        got = _run(tmp_path, tag, **env_set)
        assert got.tobytes() == default.tobytes(), tag
