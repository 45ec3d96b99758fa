"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the path at small extents.

  compute-sanitizer --tool memcheck python profiles/sanitize_case.py nano config1 c2div4
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(name):
    import torch
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import workloads as wl
    case = {"nano": wl.nano, "config1": wl.config1, "c2div4": lambda: wl.config2(div=4),
            "m3div4": lambda: wl.config2(div=4, views_rig=(1, 3))}[name]()
    m = q.Model(case.cfg, device=0)
    m.load_weights(case.store())
    rgb = m.forward_render(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams,
                           case.target)
    ldm = m.forward(case.enc_images, case.enc_cams, case.target, deltas=True)
    # device-resident path with the pipelined host frames twice
    t1 = m.submit_frame(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams,
                        case.target, np.empty_like(rgb))
    t2 = m.submit_frame(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams,
                        case.target, np.empty_like(rgb))
    m.wait_frame(t1)
    m.wait_frame(t2)
    torch.cuda.synchronize()
    print(f"{name}: rgb mean {float(rgb.mean()):.6f}, depth mean {float(ldm.depth.mean()):.4f}",
          flush=True)
    m.close()


if __name__ == "__main__":
    for n in sys.argv[1:] or ["nano", "config1"]:
        run(n)
