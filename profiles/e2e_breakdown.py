"""Where the end-to-end (host C ABI) frame time goes on config 2: wall time of
the device-input path, of the host path, and of its transfers alone."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_16680_b200 as q  # noqa: E402
from paper_2411_16680_b200 import workloads as wl  # noqa: E402


def wall(fn, n=8):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


def main():
    case = wl.config2()
    m = q.Model(case.cfg, device=0)
    m.init_weights(case.seed)
    dev = torch.device("cuda:0")
    enc_h = torch.from_numpy(case.enc_images).pin_memory()
    ren_h = torch.from_numpy(case.ren_images).pin_memory()
    plan = q.plan_forward(case.cfg, enc_h.shape[1], enc_h.shape[2])
    out_h = torch.empty((plan.out_height, plan.out_width, 3), dtype=torch.float32).pin_memory()
    enc, ren = enc_h.to(dev), ren_h.to(dev)
    rgb = torch.empty(out_h.shape, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    r = {}
    enq = []
    for _ in range(5):  # host-side enqueue cost of one frame, GPU idle at the call
        torch.cuda.synchronize()
        t = time.perf_counter()
        m.forward_render_device(enc, case.enc_cams, ren, case.ren_cams, case.target, rgb, st)
        enq.append((time.perf_counter() - t) * 1e3)
        torch.cuda.synchronize()
    r["enqueue_ms_min"] = min(enq)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(st)
    calls = []
    for _ in range(8):
        tc = time.perf_counter()
        m.forward_render_device(enc, case.enc_cams, ren, case.ren_cams, case.target, rgb, st)
        calls.append(round((time.perf_counter() - tc) * 1e3, 2))
    e1.record(st)
    torch.cuda.synchronize()
    r["device_path_event_ms"] = e0.elapsed_time(e1) / 8
    r["device_path_same_loop_wall_ms"] = (time.perf_counter() - t0) * 1e3 / 8
    r["per_call_host_ms"] = calls
    r["device_path_ms"] = wall(lambda: m.forward_render_device(enc, case.enc_cams, ren, case.ren_cams,
                                                               case.target, rgb, st))
    e_np, r_np, o_np = enc_h.numpy(), ren_h.numpy(), out_h.numpy()
    r["host_path_ms"] = wall(lambda: m.forward_render(e_np, case.enc_cams, r_np, case.ren_cams,
                                                      case.target, out=o_np))
    r["h2d_enc_ms"] = wall(lambda: enc.copy_(enc_h, non_blocking=True))
    r["h2d_ren_ms"] = wall(lambda: ren.copy_(ren_h, non_blocking=True))
    r["d2h_rgb_ms"] = wall(lambda: out_h.copy_(rgb, non_blocking=True))
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}))


if __name__ == "__main__":
    main()
