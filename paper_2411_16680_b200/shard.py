"""Multi-GPU sharding of the per-frame path.

The path partitions by independent target viewpoints (SURVEY.md §8(e),
configs 4/5): one process per GPU, rank r reconstructs and renders its own
target from the same M input views -- no data-path collective (weak
scaling). A single target can additionally be split into output row bands
(`Model.render_rows_device`, bit-identical to the full render); assembling
the bands is the one real exchange step (an all-gather of rows).

Everything here is host logic over `torch.distributed` and runs under both
NCCL (bench.py on B200s) and gloo (tests/test_multirank.py on CPU).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from .workloads import config5_targets


def target_center(rank: int, world: int) -> Tuple[float, float, float]:
    """World-space centre of rank `rank`'s target camera: the 2x4 config-5
    grid (input grid offset by half a baseline); a single process keeps the
    config-2 centre."""
    if world <= 1:
        return (0.0, 0.0, 0.0)
    grid = config5_targets()
    return grid[rank % len(grid)]


def row_band(rank: int, world: int, rows: int) -> Tuple[int, int]:
    """[r0, r1) rows of an output frame owned by `rank` (contiguous, balanced
    to within one row, covering every row exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("row_band: bad rank / world")
    return rows * rank // world, rows * (rank + 1) // world


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_fps(world: int, frames_per_rank: int, seconds_max: float) -> float:
    """Whole-job frames/s: every rank renders `frames_per_rank` frames of its
    own target; the job takes as long as its slowest rank."""
    if seconds_max <= 0:
        raise ValueError("aggregate_fps: non-positive time")
    return world * frames_per_rank / seconds_max


def gather_rows(band, rows: int, device=None):
    """All-gather the row bands of one frame ([r1 - r0, W, 3] per rank, as
    assigned by `row_band`) into the full [rows, W, 3] frame on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    width, ch = band.shape[1], band.shape[2]
    # all_gather needs equal sizes: pad every band to the largest
    hmax = max(row_band(r, world, rows)[1] - row_band(r, world, rows)[0] for r in range(world))
    pad = torch.zeros((hmax, width, ch), dtype=band.dtype, device=band.device)
    pad[: band.shape[0]] = band
    parts: List = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    out = []
    for r, p in enumerate(parts):
        r0, r1 = row_band(r, world, rows)
        out.append(p[: r1 - r0])
    return torch.cat(out, 0)


def split_counts(n: int, world: int) -> Sequence[int]:
    """Units per rank when n independent units (targets, frames) are dealt
    round-robin."""
    return [n // world + (1 if r < n % world else 0) for r in range(world)]


def view_range(rank: int, world: int, views: int) -> Tuple[int, int]:
    """[v0, v1) input views encoded by `rank` in a view-sharded encode: the
    feature pyramid is target-independent (encode_inputs, network.hpp:368-417),
    so each GPU encodes a contiguous share of the M views once per frame and
    the shares are all-gathered."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("view_range: bad rank / world")
    return views * rank // world, views * (rank + 1) // world


def allgather_views(level, views: int) -> None:
    """In-place all-gather of one pyramid level [M, H_k, W_k, C] whose view
    slices [v0, v1) (view_range) were each produced on their own rank: after
    the call every rank holds all M views. NCCL with an even split: one
    in-place all_gather_into_tensor over NVLink on the current stream; other
    backends / uneven splits: a padded all_gather."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return
    world, rank = dist.get_world_size(), dist.get_rank()
    v0, v1 = view_range(rank, world, views)
    if views % world == 0 and dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(level, level[v0:v1])
        return
    per = max(view_range(r, world, views)[1] - view_range(r, world, views)[0] for r in range(world))
    pad = torch.zeros((per,) + tuple(level.shape[1:]), dtype=level.dtype, device=level.device)
    pad[: v1 - v0] = level[v0:v1]
    parts: List = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    for r, p in enumerate(parts):
        a, b = view_range(r, world, views)
        if r != rank:
            level[a:b] = p[: b - a]
