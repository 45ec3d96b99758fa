"""The fused pyramid exchange (lvsg_pyramid_export / lvsg_pyramid_import):
two ranks, each encoding half of the views, store their pooled levels into
each other's pyramid from the conv epilogue (CUDA IPC mappings). On the one
GPU of this box both processes share the device — the kernels never wait on
each other (a host barrier orders the phases) — which checks the plumbing and
the offsets: every rank must end with the full pyramid, bit-identical to a
single-context encode, and render the same frame."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import shard
    from paper_2411_16680_b200 import workloads as wl
    try:
        dev = torch.device("cuda", 0)
        case = wl.config2(div=4)
        cfg, M, K = case.cfg, case.cfg.views, case.cfg.pyramid_levels
        enc = torch.from_numpy(case.enc_images).to(dev)
        ren = torch.from_numpy(case.ren_images).to(dev)
        He, We = enc.shape[1], enc.shape[2]
        m = q.Model(cfg, device=0)
        m.init_weights(case.seed)
        mine = m.pyramid_export((He, We))
        handles = [None] * world
        dist.all_gather_object(handles, mine)
        m.pyramid_import([h for r, h in enumerate(handles) if r != rank])
        for lv in range(K):
            m.pyramid_level(lv).fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        v0, v1 = shard.view_range(rank, world, M)
        m.encode_device(enc, v0, v1)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's stores into every pyramid have landed
        ref = q.Model(cfg, device=0)
        ref.init_weights(case.seed)
        ref.encode_device(enc)
        torch.cuda.synchronize()
        same = [bool(torch.equal(m.pyramid_level(k), ref.pyramid_level(k))) for k in range(K)]
        plan = q.plan_forward(cfg, He, We)
        a = torch.empty((plan.out_height, plan.out_width, 3), device=dev)
        b = torch.empty_like(a)
        m.forward_render_device(None, case.enc_cams, ren, case.ren_cams, case.target, a,
                                enc_hw=(He, We))
        ref.forward_render_device(enc, case.enc_cams, ren, case.ren_cams, case.target, b)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"same{rank}.npy"), np.array(same))
        np.save(os.path.join(out_dir, f"frame_eq{rank}.npy"), np.array([bool(torch.equal(a, b))]))
        dist.barrier()  # peers stop using our buffers before they are freed
        m.close()
        ref.close()
    finally:
        dist.destroy_process_group()


def test_fused_pyramid_exchange_two_ranks(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.load(tmp_path / f"same{r}.npy").all()
        assert np.load(tmp_path / f"frame_eq{r}.npy").all()
