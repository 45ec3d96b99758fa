"""Generates the committed golden fixtures in tests/golden/ from the REAL
reference (oracle/_ref/libref.so, built from /root/reference/proj by
oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Fixtures (all produced by the reference's own code paths, T=float):
  nano.npz      nano_config forward + render_target: rgb, LDM depth,
                density, blend, blend_logits, volume; FNV-1a of the weights
                and of the images
  config1.npz   BASELINE config 1 rgb (+ FNV-1a-64 of its bytes)
  stages.npz    world_points / footprint taps / gather values on random
                depths through the config-2 rig cameras
  plan.npz      plan_forward(full_scale_config, 576, 960)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import paper_2411_16680_b200 as q  # noqa: E402
from bindings import Reference, fnv1a64  # noqa: E402
from cases import config1, config2, nano  # noqa: E402

OUTS = ("rgb", "depth", "density", "blend", "blend_logits", "volume")


def main():
    ref = Reference()
    c = nano()
    w, _, _ = ref.init_param_store(c.cfg, c.seed)
    r = ref.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target, w,
                           outputs=OUTS)
    np.savez_compressed(os.path.join(HERE, "nano.npz"), **{k: r[k] for k in OUTS},
                        weights_fnv=fnv1a64(w), images_fnv=fnv1a64(c.enc_images))

    c = config1()
    w, _, _ = ref.init_param_store(c.cfg, c.seed)
    r = ref.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target, w)
    np.savez_compressed(os.path.join(HERE, "config1.npz"), rgb=r["rgb"], rgb_fnv=fnv1a64(r["rgb"]),
                        weights_fnv=fnv1a64(w), images_fnv=fnv1a64(c.enc_images))

    c = config2(div=8)
    rng = np.random.default_rng(7)
    L, H, W = 3, 45, 80
    fr = q.Frustum(c.target.camera.scaled(W, H), 0.5, 100.0)
    depth = (1.0 / rng.uniform(1 / 100.0, 1 / 0.5, size=(L, H, W))).astype(np.float32)
    pts = ref.world_points(fr, depth)
    cam = c.ren_cams[1]
    taps, valid, fracs = ref.footprints(cam, pts)
    vals, mask = ref.gather(cam, c.ren_images[1], pts)
    np.savez_compressed(os.path.join(HERE, "stages.npz"), depth=depth, points=pts, taps=taps,
                        valid=valid, fracs=fracs, values=vals, mask=mask,
                        cam=np.array(list(cam.to_c().cam_from_world) +
                                     [cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height]),
                        image_fnv=fnv1a64(c.ren_images[1]))

    p = ref.plan_forward(q.full_scale_config(), 576, 960)
    np.savez_compressed(os.path.join(HERE, "plan.npz"),
                        pyramid=np.array([[p.pyramid_h[k], p.pyramid_w[k]] for k in range(p.num_levels)]),
                        steps=np.array([[s.in_layers, s.layers, s.in_height, s.in_width, s.height,
                                         s.width, s.doubled, s.level, s.feat_h, s.feat_w,
                                         s.render_h, s.render_w, s.collapse_count]
                                        for s in list(p.steps)[:p.num_steps]]),
                        out=np.array([p.out_height, p.out_width]))
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
