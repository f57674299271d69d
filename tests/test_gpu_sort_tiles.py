"""The narrow-band sort's tile shape never changes a result: linear tiles
(`ERMC_SORT_BLOCK=0`), the default cubic tiles (the largest cube with
edge^3 R <= 2^16, clipped at the grid's faces) and an explicit small edge
give byte-identical Q_r and sigma, in fp64 and fp32, on a grid no edge
divides. The knob is read once per process, so each setting runs in its own.
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
for prec in (capi.FP64, capi.FP32):
    q, sd, st, tot, _ = capi.solve(g, t, b, m, capi.config_struct(rays_per_cell=24, seed=9,
                                                                    precision=prec))
    out += [q, sd, np.asarray(st, dtype=np.float64)]
np.save({path!r}, np.concatenate(out))
"""


def _run(tmp_path, block):
    path = str(tmp_path / f"sort_{block}.npy")
    env = dict(os.environ)
    if block is None:
        env.pop("ERMC_SORT_BLOCK", None)
    else:
        env["ERMC_SORT_BLOCK"] = str(block)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), path=path)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


def test_sort_tile_shape_never_changes_results(tmp_path):
    ref = _run(tmp_path, 0)          # linear tiles
    auto = _run(tmp_path, None)      # default: cubic, edge 13 at R = 24 (22 = 13 + 9)
    small = _run(tmp_path, 5)        # ragged 5^3 tiles
    assert ref.tobytes() == auto.tobytes()
    assert ref.tobytes() == small.tobytes()
