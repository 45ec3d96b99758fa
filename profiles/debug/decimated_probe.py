"""Steady-state ms/frame of the decimated host pipeline vs the two-resolution
one (lvsg_submit_frame[_decimated], two frames in flight), and the device
time of a decimated frame vs a regular one (CUDA events, inputs resident)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2411_16680_b200 as q
from paper_2411_16680_b200 import workloads as wl

case = wl.config2()
m = q.Model(case.cfg, device=0)
m.init_weights(case.seed)
enc_h = torch.from_numpy(case.enc_images).pin_memory().numpy()
ren_h = torch.from_numpy(case.ren_images).pin_memory().numpy()
plan = q.plan_forward(case.cfg, enc_h.shape[1], enc_h.shape[2])
outs = [torch.empty((plan.out_height, plan.out_width, 3)).pin_memory().numpy() for _ in range(2)]
He, We = enc_h.shape[1], enc_h.shape[2]


def run(dec, n=30):
    pend, t = [], []
    for k in range(n + 4):
        if len(pend) == 2:
            m.wait_frame(pend.pop(0))
        if dec:
            pend.append(m.submit_frame_decimated(ren_h, case.ren_cams, case.target, (He, We), outs[k % 2]))
        else:
            pend.append(m.submit_frame(enc_h, case.enc_cams, ren_h, case.ren_cams, case.target, outs[k % 2]))
        t.append(time.perf_counter())
    while pend:
        m.wait_frame(pend.pop(0))
    return (t[-1] - t[4]) / (len(t) - 5) * 1e3


for dec in (True, False, False, True, False, False):
    print(("decimated" if dec else "two-resolution") + f": {run(dec):.3f} ms/frame (host loop, steady state)")
m.close()
