"""Steady-state ms/frame of the view-sharded e2e pipeline (bench.py
piped_step at N=1 with --shard-encoder) with parts switched off, to find
what serialises it."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2411_16680_b200 as q  # noqa: E402
from paper_2411_16680_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda", 0)
case = wl.config2()
model = q.Model(case.cfg, device=0)
model.init_weights(case.seed)
enc_h = torch.from_numpy(case.enc_images).pin_memory()
ren_h = torch.from_numpy(case.ren_images).pin_memory()
enc = [enc_h.to(dev), enc_h.to(dev)]
ren = [ren_h.to(dev), ren_h.to(dev)]
plan = q.plan_forward(case.cfg, enc_h.shape[1], enc_h.shape[2])
rgb = [torch.empty((plan.out_height, plan.out_width, 3), device=dev) for _ in range(2)]
out = [torch.empty((plan.out_height, plan.out_width, 3)).pin_memory() for _ in range(2)]
He, We = enc_h.shape[1], enc_h.shape[2]
st, h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
up = [torch.cuda.Event(), torch.cuda.Event()]
done = [torch.cuda.Event(), torch.cuda.Event()]


def run(name, n=20, copy_in=True, copy_out=True, alt=True, split=True, what="both"):
    busy = [False, False]
    t = []
    hs = {"sync": 0.0, "enc": 0.0, "fwd": 0.0}
    for k in range(n + 4):
        s = k % 2 if alt else 0
        t0 = time.perf_counter()
        if busy[k % 2]:
            done[k % 2].synchronize()
        t1 = time.perf_counter()
        with torch.cuda.stream(h2d):
            if copy_in and what in ("both", "enc"):
                enc[s].copy_(enc_h, non_blocking=True)
            if copy_in and what in ("both", "ren"):
                ren[s].copy_(ren_h, non_blocking=True)
            up[k % 2].record(h2d)
        with torch.cuda.stream(st):
            st.wait_event(up[k % 2])
            if split:
                model.encode_device(enc[s], 0, 8, st)
                t2 = time.perf_counter()
                model.forward_render_device(None, case.enc_cams, ren[s], case.ren_cams, case.target,
                                            rgb[s], st, enc_hw=(He, We))
                t3 = time.perf_counter()
                if k >= 4:
                    hs["sync"] += t1 - t0
                    hs["enc"] += t2 - t1
                    hs["fwd"] += t3 - t2
            else:
                model.forward_render_device(enc[s], case.enc_cams, ren[s], case.ren_cams,
                                            case.target, rgb[s], st)
            d2h.wait_stream(st)
        with torch.cuda.stream(d2h):
            if copy_out:
                out[s].copy_(rgb[s], non_blocking=True)
            done[k % 2].record(d2h)
        busy[k % 2] = True
        t.append(time.perf_counter())
    for e in done:
        e.synchronize()
    dt = (t[-1] - t[4]) / (len(t) - 5) * 1e3
    print(f"{name}: {dt:.2f} ms/frame; host ms/step " +
          " ".join(f"{k} {v / n * 1e3:.2f}" for k, v in hs.items()))


run("split, copies")
run("split, copy enc only", what="enc")
run("split, copy ren only", what="ren")
run("split, no copies", copy_in=False, copy_out=False)
model.close()
