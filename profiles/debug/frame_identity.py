"""Bit-identity of one frame between two library builds (LVSG_LIB) on a
workload: python profiles/debug/frame_identity.py <lib_a> <lib_b> [case]."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
RUN = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + '/tests']
import paper_2411_16680_b200 as q
from paper_2411_16680_b200 import workloads as wl
case = {'c2div4': lambda: wl.config2(div=4), 'c2': lambda: wl.config2(), 'config1': wl.config1}[sys.argv[2]]()
m = q.Model(case.cfg, device=0)
m.load_weights(case.store())
np.save(sys.argv[3], m.forward_render(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams, case.target))
"""
case = sys.argv[3] if len(sys.argv) > 3 else "c2div4"
outs = []
for i, lib in enumerate(sys.argv[1:3]):
    env = dict(os.environ, LVSG_LIB=lib)
    path = f"/tmp/fi_{i}.npy"
    subprocess.run([sys.executable, "-c", RUN, ROOT, case, path], env=env, check=True)
    outs.append(np.load(path))
same = np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
print(f"{case}: bit-identical {same}, max-abs {float(np.abs(outs[0] - outs[1]).max()):.3e}")
