"""In-pipeline timeline of a config-2 frame's conv launches (PDL on, nothing
serialised): globaltimer at each launch's first CTA entry, at its grid
dependency wait returning, and at its last CTA exit. Needs the LVSG_TIMELINE
build:
  bash profiles/debug/build_variant.sh tl "-DLVSG_TIMELINE=1"
  LVSG_LIB=build/variant/tl/liblvsg.so python profiles/debug/conv_timeline.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2411_16680_b200 as q  # noqa: E402
from paper_2411_16680_b200 import workloads as wl  # noqa: E402

case = wl.config2()
dev = torch.device("cuda", 0)
model = q.Model(case.cfg, device=0)
model.init_weights(case.seed)
enc = torch.from_numpy(case.enc_images).to(dev)
ren = torch.from_numpy(case.ren_images).to(dev)
plan = q.plan_forward(case.cfg, enc.shape[1], enc.shape[2])
rgb = torch.empty((plan.out_height, plan.out_width, 3), device=dev)
st = torch.cuda.Stream()
lib = model._lib
fn = lib.lvsg_debug_conv_timeline
fn.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32)]
n = ctypes.c_int32(0)


def frame():
    with torch.cuda.stream(st):
        model.forward_render_device(enc, case.enc_cams, ren, case.ren_cams, case.target, rgb, st)


for _ in range(3):
    frame()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fn(model._h, 0, None, ctypes.byref(n))
e0.record(st)
frame()
e1.record(st)
buf = np.zeros((1024, 4), dtype=np.uint64)
n.value = 1024
fn(model._h, 1, buf.ctypes.data, ctypes.byref(n))
fn(model._h, 2, None, ctypes.byref(n))
torch.cuda.synchronize()
k = n.value
if k < 0:
    raise SystemExit("not an LVSG_TIMELINE build")
valid = buf[:k, 3] > 0  # launches that ran the tensor-core kernel
base = int(buf[:k][valid, 0].min())
t = np.zeros((k, 4))
for i in range(k):
    if valid[i]:
        t[i, :3] = (buf[i, :3].astype(np.int64) - base).astype(np.float64)
        t[i, 3] = float(buf[i, 3])
np.save("gpurun_out/conv_timeline.npy", buf[:k])
base = 0.0
print(f"frame {e0.elapsed_time(e1):.3f} ms (events), {k} conv launches")
print("  #   entry   ready    exit  run(ready->exit)  wait(entry->ready)  gap(prev exit->ready)  CTAs")
tot_run = 0.0
small = [0, 0.0]
prev_ex = None
for i in range(k):
    if not valid[i]:
        print(f"{i:3d}  (not a tensor-core launch)")
        continue
    en, rd, ex, ctas = (t[i, 0] - base) / 1e3, (t[i, 1] - base) / 1e3, (t[i, 2] - base) / 1e3, int(t[i, 3])
    gap = rd - prev_ex if prev_ex is not None else 0.0
    prev_ex = ex
    run = ex - rd
    tot_run += run
    if run < 20:
        small[0] += 1
        small[1] += run
    print(f"{i:3d} {en:8.1f} {rd:8.1f} {ex:8.1f} {run:10.1f} {rd - en:14.1f} {gap:14.1f} {ctas:6d}")
print(f"sum of run times {tot_run:.1f} us; launches under 20 us: {small[0]}, {small[1]:.1f} us")
model.close()
