"""Throughput on BASELINE.json's other configs, one B200 (device-timed with
CUDA events on the frame stream, L2 flushed between frames; host-pipelined
e2e where it applies). Prints one JSON line per config.

  config3: 16 views of 1080p (576x960 encoder), one target
  config4: the 30-frame video: per-frame inputs (moving scene) and a moving
           target, every frame a full reconstruct + render; device and e2e
           (lvsg_submit_frame, two frames in flight)
  config5: 8 target viewpoints of one frame: one encode (lvsg_encode_device)
           + 8 forward-renders from the resident pyramid, against 8 full
           forward-renders
"""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _frame(t):
    from paper_2411_16680_b200 import workloads as wl
    c = wl.config4_frame(t)
    return c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target


def timed(stream, flush, fn, n):
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(n)]
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for k in range(n):
            flush.zero_()
            ev[k][0].record(stream)
            fn(k)
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / n


def main(which=("config3", "config4", "config5")):
    import torch
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import workloads as wl
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    if "config3" in which:
        c = wl.config3()
        m = q.Model(c.cfg, device=0)
        m.init_weights(c.seed)
        enc = torch.from_numpy(c.enc_images).to(dev)
        ren = torch.from_numpy(c.ren_images).to(dev)
        p = q.plan_forward(c.cfg, enc.shape[1], enc.shape[2])
        rgb = torch.empty((p.out_height, p.out_width, 3), device=dev)
        f = lambda k: m.forward_render_device(enc, c.enc_cams, ren, c.ren_cams, c.target, rgb, stream)  # noqa: E731
        for _ in range(3):
            f(0)
        ms = timed(stream, flush, f, 10)
        print(json.dumps({"config": "config3: 16 views, 576x960 -> 1080p", "ms_per_frame": ms,
                          "frames_per_s": 1000.0 / ms}), flush=True)
        m.close()
        del enc, ren

    if "config4" in which:
        with ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
            frames = list(ex.map(_frame, range(30)))
        c0 = wl.config4_frame(0)
        m = q.Model(c0.cfg, device=0)
        m.init_weights(c0.seed)
        encs = [torch.from_numpy(f[0]).to(dev) for f in frames]
        rens = [torch.from_numpy(f[2]).to(dev) for f in frames]
        p = q.plan_forward(c0.cfg, encs[0].shape[1], encs[0].shape[2])
        rgb = torch.empty((p.out_height, p.out_width, 3), device=dev)

        def f(k):
            e, ec, r, rc, tg = frames[k % 30]
            m.forward_render_device(encs[k % 30], ec, rens[k % 30], rc, tg, rgb, stream)
        for k in range(3):
            f(k)
        ms = timed(stream, flush, f, 30)
        del encs, rens
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
        hosts = [(pin(f[0]), f[1], pin(f[2]), f[3], f[4]) for f in frames]
        outs = [pin(torch.zeros((p.out_height, p.out_width, 3)).numpy()) for _ in range(2)]
        pend = []
        for k in range(3):  # warm both frame slots
            e, ec, r, rc, tg = hosts[k]
            pend.append(m.submit_frame(e, ec, r, rc, tg, outs[k % 2]))
            if len(pend) == 2:
                m.wait_frame(pend.pop(0))
        while pend:
            m.wait_frame(pend.pop(0))
        t0 = time.perf_counter()
        for k in range(30):
            if len(pend) == 2:
                m.wait_frame(pend.pop(0))
            e, ec, r, rc, tg = hosts[k]
            pend.append(m.submit_frame(e, ec, r, rc, tg, outs[k % 2]))
        while pend:
            m.wait_frame(pend.pop(0))
        e2e = 30.0 / (time.perf_counter() - t0)
        print(json.dumps({"config": "config4: 30-frame video, moving scene and target, 8 views, "
                                    "per-frame LDM re-creation", "ms_per_frame": ms,
                          "frames_per_s": 1000.0 / ms, "e2e_frames_per_s": e2e,
                          "e2e_path": "lvsg_submit_frame / lvsg_wait_frame, pinned host frames"}),
              flush=True)
        m.close()

    if "config5" in which:
        c = wl.config2()
        m = q.Model(c.cfg, device=0)
        m.init_weights(c.seed)
        enc = torch.from_numpy(c.enc_images).to(dev)
        ren = torch.from_numpy(c.ren_images).to(dev)
        He, We = enc.shape[1], enc.shape[2]
        p = q.plan_forward(c.cfg, He, We)
        rgb = torch.empty((p.out_height, p.out_width, 3), device=dev)
        # the config-5 grid: the 2x4 input grid offset by half a baseline
        tg_full = [q.Frustum(wl._target_cam(1920, 1080, 1080.0, ctr), 0.5, 100.0)
                   for ctr in wl.config5_targets()]

        def shared(k):
            m.encode_device(enc, 0, c.cfg.views, stream)
            for tg in tg_full:
                m.forward_render_device(None, c.enc_cams, ren, c.ren_cams, tg, rgb, stream,
                                        enc_hw=(He, We))

        def separate(k):
            for tg in tg_full:
                m.forward_render_device(enc, c.enc_cams, ren, c.ren_cams, tg, rgb, stream)
        for _ in range(2):
            shared(0)
            separate(0)
        ms_sh = timed(stream, flush, shared, 5)
        ms_sep = timed(stream, flush, separate, 5)
        print(json.dumps({"config": "config5: 8 target viewpoints of one frame (8 views)",
                          "ms_per_8_targets_one_encode": ms_sh,
                          "target_frames_per_s_one_encode": 8000.0 / ms_sh,
                          "ms_per_8_targets_separate": ms_sep,
                          "target_frames_per_s_separate": 8000.0 / ms_sep}), flush=True)
        m.close()


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or ("config3", "config4", "config5"))
