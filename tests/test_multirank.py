"""The N > 1 host path on CPU: world_size-2 gloo process groups exercising
paper_2411_16680_b200.shard (target sharding, row bands, max-over-ranks
timing, band all-gather), with the oracle as each rank's renderer."""
import os
import socket

import numpy as np
import pytest

from paper_2411_16680_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
        from bindings import Oracle
        from paper_2411_16680_b200 import workloads as wl

        # (1) target sharding: each rank renders its own viewpoint of the same inputs
        center = shard.target_center(rank, world)
        case = wl.config2(div=4, target_center=center)
        o = Oracle()
        rgb = o.forward_render(case.cfg, case.enc_images, case.enc_cams, case.ren_images,
                               case.ren_cams, case.target, case.flat())["rgb"]
        np.save(os.path.join(out_dir, f"rgb{rank}.npy"), rgb)

        # (2) timing = the slowest rank
        slowest = shard.max_over_ranks(1.0 + rank)
        fps = shard.aggregate_fps(world, 3, slowest)

        # (3) one target split into row bands and re-assembled by all-gather
        full = o.forward_render(*_center_case())["rgb"]
        rows = full.shape[0]
        r0, r1 = shard.row_band(rank, world, rows)
        frame = shard.gather_rows(torch.from_numpy(np.ascontiguousarray(full[r0:r1])), rows)
        np.save(os.path.join(out_dir, f"gathered{rank}.npy"), frame.numpy())
        np.save(os.path.join(out_dir, f"full{rank}.npy"), full)
        with open(os.path.join(out_dir, f"t{rank}.txt"), "w") as f:
            f.write(f"{slowest} {fps}")

        # (4) view-sharded encode: rank r produces pyramid views view_range(r)
        # (here a deterministic stand-in per view), the all-gather completes
        # every rank's copy; even (M=4) and uneven (M=5) splits
        for M in (4, 5):
            full_lv = torch.arange(M * 3 * 5 * 8, dtype=torch.float32).reshape(M, 3, 5, 8)
            mine = torch.full_like(full_lv, float("nan"))
            v0, v1 = shard.view_range(rank, world, M)
            mine[v0:v1] = full_lv[v0:v1]
            shard.allgather_views(mine, M)
            np.save(os.path.join(out_dir, f"pyr{M}_{rank}.npy"), mine.numpy())
    finally:
        dist.destroy_process_group()


def _center_case():
    from paper_2411_16680_b200 import workloads as wl
    c = wl.nano()
    return (c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target, c.flat())


def test_row_bands_partition_rows():
    for world in (1, 2, 3, 8):
        for rows in (1, 7, 64, 1080):
            if world > rows:
                continue
            bands = [shard.row_band(r, world, rows) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
            sizes = [b - a for a, b in bands]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.row_band(2, 2, 10)
    assert list(shard.split_counts(10, 4)) == [3, 3, 2, 2]


def test_targets_distinct_per_rank():
    assert shard.target_center(0, 1) == (0.0, 0.0, 0.0)
    cs = [shard.target_center(r, 8) for r in range(8)]
    assert len(set(cs)) == 8


def test_two_rank_gloo(oracle, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    a, b = (np.load(tmp_path / f"rgb{r}.npy") for r in range(world))
    assert a.shape == b.shape
    assert not np.array_equal(a, b)  # distinct target viewpoints
    for r in range(world):
        slowest, fps = map(float, open(tmp_path / f"t{r}.txt").read().split())
        assert slowest == 2.0 and abs(fps - world * 3 / 2.0) < 1e-12
        g = np.load(tmp_path / f"gathered{r}.npy")
        assert np.array_equal(g, np.load(tmp_path / f"full{r}.npy"))
        for M in (4, 5):
            want = np.arange(M * 3 * 5 * 8, dtype=np.float32).reshape(M, 3, 5, 8)
            assert np.array_equal(np.load(tmp_path / f"pyr{M}_{r}.npy"), want)


def test_view_ranges_partition_views():
    for world in (1, 2, 4, 8):
        for views in (8, 16, 5):
            rs = [shard.view_range(r, world, views) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == views
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
