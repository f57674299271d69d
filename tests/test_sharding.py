"""Multi-rank path on CPU: world_size-2 gloo processes each solve their
x-slab and assemble Q_r with the same all-gather the GPU ranks use (NCCL on
the box). The per-rank solver here is the C oracle standing in for the GPU
(test-only); the product's solve_range bitwise-slab property is covered by
tests/test_gpu_parity.py::test_slab_ranges_reassemble_bitwise.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent

from paper_1810_00188_b200 import parallel  # noqa: E402


@pytest.mark.parametrize("nx,world", [(8, 2), (7, 2), (16, 3), (5, 5), (256, 8)])
def test_x_slabs_tile_the_grid(nx, world):
    parallel.check_partition(nx, 3, 4, world)
    slabs = parallel.all_slabs(nx, 3, 4, world)
    assert max(s.n for s in slabs) - min(s.n for s in slabs) <= 12
    assert all(s.lo % 12 == 0 for s in slabs)  # whole x-planes


def _worker(rank, world, port, name, result_path):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle"), str(ROOT / "tests")]
    import oracle  # noqa: PLC0415
    from helpers import load_golden_solve  # noqa: PLC0415

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, t, b, m, c, _ = load_golden_solve(name)

    def solve_slab(slab):
        q, sd, steps, _ = oracle.solve(g, t, b, m, c, cell_range=(slab.lo, slab.hi), threads=1)
        return torch.from_numpy(q), torch.from_numpy(sd), torch.from_numpy(steps.copy())

    q, sd, steps = parallel.solve_sharded(solve_slab, g.nx, g.ny, g.nz, dist)
    if rank == 0:
        np.savez(result_path, q=q.numpy(), sd=sd.numpy(), steps=steps.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["nb_parab_6", "epsw_low_6"])
def test_two_rank_gloo_assembly_is_bitwise(tmp_path, name):
    sys.path[:0] = [str(ROOT / "tests")]
    from helpers import load_golden_solve  # noqa: PLC0415

    port = 29500 + (os.getpid() % 1000)
    out = tmp_path / "r.npz"
    mp.spawn(_worker, args=(2, port, name, str(out)), nprocs=2, join=True)
    r = np.load(out)
    *_, e = load_golden_solve(name)
    assert np.array_equal(r["q"], e["q_r"])
    assert np.array_equal(r["sd"], e["std_dev"])
    assert list(r["steps"]) == list(e["steps"])
