"""Multi-rank paths on the GPU box (ranks share its one GPU; gloo carries the
handles and barriers, CUDA IPC the data):

* the fused reduce + all-gather (session_solve_scatter): every rank's
  full-field buffer equals a one-GPU solve byte for byte;
* bench.py's N > 1 flow under torchrun (fused gather and NCCL-style slabs).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _torchrun(n, args, port, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port)] + args
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                          env=dict(os.environ, **(env or {})))


@pytest.mark.parametrize("world,precision", [(2, "fp64"), (3, "fp32")])
def test_fused_gather_is_byte_identical(world, precision):
    r = _torchrun(world, ["tools/fused_gather_check.py", "--precision", precision],
                  29600 + world)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert all(line["byte_identical_on_every_rank"])


@pytest.mark.parametrize("gather", ["fused", "nccl"])
def test_bench_multirank_flow(gather):
    r = _torchrun(2, ["bench.py", "--gpus", "2", "--steps", "1", "--warmup", "1", "--grid", "64",
                      "--rays", "8", "--no-e2e", "--no-cpu"],
                  29610 + (gather == "fused"),
                  env={"ERMC_BENCH_BACKEND": "gloo", "ERMC_BENCH_GATHER": gather})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0
    assert (lines[0]["gather"] == "fused") == (gather == "fused")


@pytest.mark.parametrize("gather", ["fused", "nccl"])
def test_bench_gpus_flag_spawns_ranks_without_torchrun(gather):
    # `python bench.py --gpus 2` exactly as written (no launcher): bench.py
    # starts both ranks itself. On this one-GPU box they share the device,
    # so the collectives switch to gloo by themselves.
    env = dict(os.environ, ERMC_BENCH_GATHER=gather)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "ERMC_BENCH_BACKEND"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--grid", "48", "--rays", "8", "--no-fp32-extra", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["ranks_share_gpu"] is True
    assert line["backend"] == "gloo"
    assert line["gather"] == ("fused" if gather == "fused" else "all-gather")
    assert line["e2e"]["value"] > 0


def test_bench_reference_arm_under_torchrun_prints_once():
    r = _torchrun(2, ["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                      "--warmup", "0", "--grid", "32", "--no-single-worker"], 29620)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
