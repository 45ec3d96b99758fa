"""Where the GPU frame differs from the oracle on a config (default: config 3
at full scale): error histogram of the RGB frame and of the LDM maps
(depth, density, blend), and the LDM error at the worst RGB pixels. Prints
one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main(name="config3"):
    import paper_2411_16680_b200 as q
    from paper_2411_16680_b200 import workloads as wl
    from bindings import Oracle
    case = wl.config3(div=1) if name == "config3" else wl.config2(div=1)
    m = q.Model(case.cfg, device=0)
    m.load_weights(case.store())
    rgb = m.forward_render(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams,
                           case.target)
    ldm = m.forward(case.enc_images, case.enc_cams, case.target)
    want = Oracle().forward_render(case.cfg, case.enc_images, case.enc_cams, case.ren_images,
                                   case.ren_cams, case.target, case.flat(),
                                   outputs=("rgb", "depth", "density", "blend"))
    d = np.abs(rgb - want["rgb"]).max(-1)
    out = {"case": case.name, "rgb_max_abs": float(d.max()),
           "rgb_px_gt_1e-5": int((d > 1e-5).sum()), "rgb_px_gt_1e-4": int((d > 1e-4).sum()),
           "rgb_px": int(d.size)}
    for k in ("depth", "density", "blend"):
        g, w = getattr(ldm, k), want[k]
        out[f"{k}_max_rel"] = float((np.abs(g - w) / np.maximum(np.abs(w), 1e-6)).max())
    idx = np.argsort(d.ravel())[-5:]
    worst = []
    for f in idx:
        i, j = divmod(int(f), d.shape[1])
        dd = np.abs(ldm.depth[:, i, j] - want["depth"][:, i, j]).max()
        bb = np.abs(ldm.blend[:, i, j] - want["blend"][:, i, j]).max()
        worst.append({"px": [i, j], "rgb": float(d[i, j]), "depth_abs": float(dd),
                      "blend_abs": float(bb)})
    out["worst"] = worst
    print(json.dumps(out))
    m.close()


if __name__ == "__main__":
    main(*sys.argv[1:])
