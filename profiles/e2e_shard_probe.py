"""Wall-clock breakdown of the view-sharded e2e step at N=1 (bench.py
--shard-encoder): where the time goes between the encoder-share upload, the
encode, and the NULL-encoder host C ABI call. Prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import workloads as wl
    dev = torch.device("cuda", 0)
    case = wl.config2()
    cfg = case.cfg
    M = cfg.views
    m = q.Model(cfg, device=0)
    m.init_weights(case.seed)
    enc_h = torch.from_numpy(case.enc_images).pin_memory()
    ren_h = torch.from_numpy(case.ren_images).pin_memory()
    enc = enc_h.to(dev)
    He, We = enc.shape[1], enc.shape[2]
    plan = q.plan_forward(cfg, He, We)
    out_h = torch.empty((plan.out_height, plan.out_width, 3)).pin_memory()
    r_np, o_np = ren_h.numpy(), out_h.numpy()
    cs = torch.cuda.ExternalStream(m.stream_handle(), device=dev)
    res = {}

    def timed(name, fn, n=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0) / n * 1e3

    def up_encode():
        with torch.cuda.stream(cs):
            enc.copy_(enc_h, non_blocking=True)
            m.encode_device(enc, 0, M, cs)
        cs.synchronize()

    def fr_null():
        m.forward_render(None, case.enc_cams, r_np, case.ren_cams, case.target, out=o_np,
                         enc_hw=(He, We))

    def both():
        with torch.cuda.stream(cs):
            enc.copy_(enc_h, non_blocking=True)
            m.encode_device(enc, 0, M, cs)
        fr_null()

    def full():
        m.forward_render(enc_h.numpy(), case.enc_cams, r_np, case.ren_cams, case.target, out=o_np)

    def both_sync():
        up_encode()
        fr_null()

    timed("upload+encode_ms", up_encode)
    timed("sharded_step_synced_ms", both_sync)
    timed("forward_render_null_ms", fr_null)
    timed("sharded_step_ms", both)
    timed("host_abi_full_ms", full)
    print(json.dumps(res))
    torch.cuda.synchronize()
    m.close()


if __name__ == "__main__":
    main()
