"""Multi-GPU partitioning of the solve.

ERMC cells are independent units: a cell's Q_r depends only on its own rays,
which read the replicated temperature field. Ranks (one process per GPU)
therefore own contiguous x-slabs of linear cell ids — the reference's worker
chunks (solver.cpp:163-167) — with no data-path exchange. The only
collectives are the assembly of the solution: an all-gather of the q_r /
std_dev slabs (NCCL over NVLink on B200s) and a sum of the step counters.
Because each cell is computed identically wherever it runs, the assembled
field is byte-identical for any GPU count (the GPU analogue of P8).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    lo: int  # first linear cell (inclusive)
    hi: int  # last linear cell (exclusive)

    @property
    def n(self) -> int:
        return self.hi - self.lo


def x_slab(nx: int, ny: int, nz: int, world: int, rank: int) -> Slab:
    """Contiguous x-planes for `rank`: planes [rank*nx/world, (rank+1)*nx/world)
    (balanced to within one plane)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    plane = ny * nz
    p0 = (rank * nx) // world
    p1 = ((rank + 1) * nx) // world
    return Slab(rank, world, p0 * plane, p1 * plane)


def all_slabs(nx: int, ny: int, nz: int, world: int) -> list[Slab]:
    return [x_slab(nx, ny, nz, world, r) for r in range(world)]


def max_slab_cells(nx: int, ny: int, nz: int, world: int) -> int:
    return max(s.n for s in all_slabs(nx, ny, nz, world))


def gather_slabs(local, slabs: list[Slab], dist, group=None):
    """All-gathers per-rank slabs (torch tensors, 1-D, this rank's cells) into
    the full field on every rank. Slabs may differ by one plane: each rank
    pads to the largest slab and the padding is dropped after the gather."""
    import torch  # noqa: PLC0415

    width = max(s.n for s in slabs)
    # NCCL gathers device tensors in place; gloo (CPU tests) through the host.
    staged = local.is_cuda and dist.get_backend(group) != "nccl"
    src = local.cpu() if staged else local
    buf = src.new_zeros(width)
    buf[: src.numel()] = src
    out = src.new_zeros(width * len(slabs))
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = [out[r * width: r * width + s.n] for r, s in enumerate(slabs)]
    full = torch.cat(parts)
    return full.to(local.device) if staged else full


def sum_counters(steps, dist, group=None):
    """Sum of the per-level step counters over ranks (int64)."""
    dist.all_reduce(steps, op=dist.ReduceOp.SUM, group=group)
    return steps


def solve_sharded(solve_slab: Callable[[Slab], tuple], nx: int, ny: int, nz: int, dist,
                  device=None):
    """Generic driver: this rank solves its slab with `solve_slab(slab)` ->
    (q_slab, sd_slab, steps_per_level) as torch tensors on `device`, then the
    slabs are assembled on every rank. Returns (q_r, std_dev, steps)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    slabs = all_slabs(nx, ny, nz, world)
    q, sd, steps = solve_slab(slabs[rank])
    q_all = gather_slabs(q, slabs, dist)
    sd_all = gather_slabs(sd, slabs, dist)
    steps = sum_counters(steps, dist)
    return q_all, sd_all, steps


def check_partition(nx: int, ny: int, nz: int, world: int) -> None:
    slabs = all_slabs(nx, ny, nz, world)
    cover = np.zeros(nx * ny * nz, dtype=np.int32)
    for s in slabs:
        cover[s.lo:s.hi] += 1
    if not np.all(cover == 1):
        raise AssertionError("slabs do not tile the grid")
