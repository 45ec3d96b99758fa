"""Deterministic synthetic workloads for every BASELINE config (SURVEY.md
§8(d)): reference camera rigs, make_scene + oracle_render images and
init_param_store weights, all from the native host generator (bit-identical
to the reference's own generator; tests/test_host.py pins that).

  config1()          4 views 256^2, C=32, Bp + 2 U&F steps (CPU-oracle case)
  config2(div=1)     8 views, full_scale_config, encoder 576x960, render 1080p
  config2(div=4)     same schedule at 1/4 extents (the bounded CPU sample)
  config3()          16 views (4x4 rig, 0.15 m baseline), across-view stress
  config4_frame(t)   frame t of the 30-frame dynamic video
  config5_targets()  8 target viewpoints (2x4 grid offset half a baseline)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import List

import numpy as np

from .camera import Camera, Frustum, RigSpec, pose_cam_from_world
from .config import ModelConfig, config1 as _cfg1, full_scale_config, micro_config, nano_config, \
    scaled_full_config
from .lvs import init_param_store, rig_cameras, scene_images


@dataclass
class Case:
    name: str
    cfg: ModelConfig
    enc_images: np.ndarray
    enc_cams: List[Camera]
    ren_images: np.ndarray
    ren_cams: List[Camera]
    target: Frustum
    seed: int = 3

    def store(self):
        return init_param_store(self.cfg, self.seed)

    def flat(self):
        return init_param_store(self.cfg, self.seed, flat=True)


def _rig_case(name, cfg, rig, tgt_cam, near, far, render_hw=None, scene_seed=21, planes=3):
    cams, _ = rig_cameras(rig)
    target = Frustum(tgt_cam, near, far)
    imgs = scene_images(scene_seed, planes, target, cams)
    if render_hw is None:
        return Case(name, cfg, imgs, cams, imgs, cams, target)
    Hr, Wr = render_hw
    rcams = [c.scaled(Wr, Hr) for c in cams]
    rimgs = scene_images(scene_seed, planes, target, rcams)
    return Case(name, cfg, imgs, cams, rimgs, rcams, target)


def nano(**ablate) -> Case:
    cfg = replace(nano_config(), **ablate)
    return _rig_case("nano" + "".join("_" + k for k in ablate), cfg,
                     RigSpec(2, 2, 0.05, 64, 64, 64.0), Camera.make(64, 64, 32, 32, 64, 64),
                     1.0, 6.0)


def nano_two_res() -> Case:
    """Encoder at 64x64, render images at 96x128 (anisotropic re-digitisation,
    the config-2 plumbing of SURVEY.md §0)."""
    return _rig_case("nano_two_res", nano_config(), RigSpec(2, 2, 0.05, 64, 64, 64.0),
                     Camera.make(64, 64, 32, 32, 64, 64), 1.0, 6.0, render_hw=(96, 128))


def micro() -> Case:
    """tests/test_network.cpp:19-40 (2 views 16x16, C=4)."""
    return _rig_case("micro", micro_config(), RigSpec(1, 2, 0.05, 16, 16, 12.0),
                     Camera.make(20.0, 20.0, 8.0, 8.0, 16, 16), 1.0, 5.0)


def config1() -> Case:
    return _rig_case("config1", _cfg1(), RigSpec(2, 2, 0.1, 256, 256, 256.0),
                     Camera.make(256, 256, 128, 128, 256, 256), 1.0, 20.0)


def _target_cam(w, h, focal, center=(0.0, 0.0, 0.0)):
    if tuple(center) == (0.0, 0.0, 0.0):  # RigSpec::target(): identity pose
        return Camera.make(focal, focal, w / 2.0, h / 2.0, w, h, np.eye(4))
    return Camera.make(focal, focal, w / 2.0, h / 2.0, w, h,
                       pose_cam_from_world(np.eye(3), center))


def config2(div: int = 1, views_rig=(2, 4), baseline=0.1, target_center=(0.0, 0.0, 0.0),
            scene_shift=0.0, scene_frustum=None) -> Case:
    """8 views of the 2x4 rig (0.3 m span), full_scale_config, encoder images
    576x960 (the same cameras .scaled), render images 1080x1920, target at
    `target_center` (rig centroid by default), near 0.5, far 100.
    div > 1: same schedule, every extent / div."""
    rows, cols = views_rig
    cfg = full_scale_config() if div == 1 else scaled_full_config(div)
    cfg = replace(cfg, views=rows * cols)
    Hr, Wr = 1080 // div, 1920 // div
    He, We = 576 // div, 960 // div
    focal = 1080.0 / div
    rcams, _ = rig_cameras(RigSpec(rows, cols, baseline, Wr, Hr, focal))
    target = Frustum(_target_cam(Wr, Hr, focal, target_center), 0.5, 100.0)
    scene_fr = scene_frustum or Frustum(_target_cam(Wr, Hr, focal), 0.5, 100.0)
    ecams = [c.scaled(We, He) for c in rcams]
    if scene_shift:
        eimgs = _shifted_scene_images(scene_fr, ecams, scene_shift)
        rimgs = _shifted_scene_images(scene_fr, rcams, scene_shift)
    else:
        eimgs = scene_images(21, 3, scene_fr, ecams)
        rimgs = scene_images(21, 3, scene_fr, rcams)
    return Case(f"config2_div{div}_m{rows * cols}", cfg, eimgs, ecams, rimgs, rcams, target)


def config3(div: int = 1) -> Case:
    """16 views, 4x4 rig with 0.15 m baseline (0.45 m span)."""
    c = config2(div=div, views_rig=(4, 4), baseline=0.15)
    c.name = f"config3_div{div}"
    return c


def _shifted_scene_images(scene_fr, cams, shift):
    # Config 4's dynamic content: make_scene(21, 3) with
    # every plane except the backdrop wall shifted by `shift` metres along x.
    return scene_images(21, 3, scene_fr, cams, shift_x=shift)


def config4_frame(t: int, div: int = 1) -> Case:
    """Frame t of the 30-frame video: target centre (0.15 sin 2pi t/30,
    0.05 cos 2pi t/30, 0) looking +z, content shifted 0.005 t m."""
    ctr = (0.15 * math.sin(2 * math.pi * t / 30.0), 0.05 * math.cos(2 * math.pi * t / 30.0), 0.0)
    c = config2(div=div, target_center=ctr, scene_shift=0.005 * t)
    c.name = f"config4_t{t}_div{div}"
    return c


def config5_targets(div: int = 1):
    """8 target viewpoints: the 2x4 input grid offset by half a baseline."""
    out = []
    for r in range(2):
        for c in range(4):
            x = (c - 1.5) * 0.1 + 0.05
            y = (r - 0.5) * 0.1 + 0.05
            out.append((x, y, 0.0))
    return out
