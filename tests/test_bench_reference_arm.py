"""bench.py's reference arm (CPU; no GPU needed): it runs the unmodified
reference's own `_ermc` module (oracle/_ref) on inputs built with the
reference's own builders, maps no shared library of this package, and
reports a config identical to the GPU arm's — including the FNV-1a hashes
of the TFLD1 / KTAB1 bytes, which each arm writes with its own writers."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

import refshim
from paper_1810_00188_b200 import workloads as W

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")

PROBE = """
import json, runpy, sys
sys.argv = ['bench.py', '--impl', 'reference', '--grid', '{n}', '--rays', '16', '--steps', '1',
            '--warmup', '0', '--no-single-worker', '--model', '{model}']
runpy.run_path('bench.py', run_name='__main__')
maps = open('/proc/self/maps').read().splitlines()
print('MAPS ' + json.dumps(sorted({{l.split()[-1] for l in maps if '{root}' in l}})))
"""


@pytest.mark.parametrize("model", ["nongrey16", "grey"])
def test_reference_arm_is_reference_only_and_same_config(model):
    n = 16
    r = subprocess.run([sys.executable, "-c", PROBE.format(n=n, model=model, root=ROOT)],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    maps = json.loads([x for x in r.stdout.splitlines() if x.startswith("MAPS ")][0][5:])
    assert maps and all("/oracle/_ref/" in m for m in maps), maps
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    _, t, _, _, m_obj = W.channel_case(n, model)
    hashes = W.file_hashes(n, t, m_obj)
    assert line["config"]["tfld_fnv"] == hashes["tfld_fnv"]
    assert line["config"]["ktab_fnv"] == hashes["ktab_fnv"]
    sys.path.insert(0, str(ROOT))
    import bench  # noqa: PLC0415

    class A:  # the GPU arm's argument namespace for the same workload
        grid, rays, model_, precision, seed, wall_eps = n, 16, model, "fp64", 2024, 1.0
    a = A()
    a.model = model
    assert line["config"] == bench.config_dict(a, 1, hashes)


def test_gpus_flag_spawns_ranks_without_a_launcher():
    # `bench.py --gpus 2` with no WORLD_SIZE: bench.py starts both ranks
    # itself (the driver's N > 1 invocation works with or without torchrun);
    # on the reference arm rank 0 alone runs and prints one line.
    import os
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                        "--grid", "16", "--rays", "8", "--steps", "1", "--warmup", "0",
                        "--no-single-worker"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
