"""Deterministic synthetic cases shared by the parity tests and the bench
(SURVEY.md §8(d)): reference rigs, make_scene + oracle_render images and
init_param_store weights, all produced by the product's host generator
(bit-identical to the reference's; tests/test_host.py pins that)."""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import List

import numpy as np

import paper_2411_16680_b200 as q


@dataclass
class Case:
    name: str
    cfg: q.ModelConfig
    enc_images: np.ndarray
    enc_cams: List[q.Camera]
    ren_images: np.ndarray
    ren_cams: List[q.Camera]
    target: q.Frustum
    seed: int = 3

    def store(self):
        return q.init_param_store(self.cfg, self.seed)

    def flat(self):
        return q.init_param_store(self.cfg, self.seed, flat=True)


def _rig_case(name, cfg, rig, tgt_cam, near, far, render_hw=None, scene_seed=21, planes=3):
    cams, _ = q.rig_cameras(rig)
    target = q.Frustum(tgt_cam, near, far)
    imgs = q.scene_images(scene_seed, planes, target, cams)
    if render_hw is None:
        return Case(name, cfg, imgs, cams, imgs, cams, target)
    Hr, Wr = render_hw
    rcams = [c.scaled(Wr, Hr) for c in cams]
    rimgs = q.scene_images(scene_seed, planes, target, rcams)
    return Case(name, cfg, imgs, cams, rimgs, rcams, target)


def nano(**ablate) -> Case:
    cfg = replace(q.nano_config(), **ablate)
    return _rig_case("nano" + "".join("_" + k for k in ablate), cfg,
                     q.RigSpec(2, 2, 0.05, 64, 64, 64.0), q.Camera.make(64, 64, 32, 32, 64, 64),
                     1.0, 6.0)


def nano_two_res() -> Case:
    """Encoder at 64x64, render images at 96x128 (anisotropic re-digitisation,
    the config-2 plumbing of SURVEY.md §0)."""
    return _rig_case("nano_two_res", q.nano_config(), q.RigSpec(2, 2, 0.05, 64, 64, 64.0),
                     q.Camera.make(64, 64, 32, 32, 64, 64), 1.0, 6.0, render_hw=(96, 128))


def micro() -> Case:
    """tests/test_network.cpp:19-40 (2 views 16x16, C=4)."""
    return _rig_case("micro", q.micro_config(), q.RigSpec(1, 2, 0.05, 16, 16, 12.0),
                     q.Camera.make(20.0, 20.0, 8.0, 8.0, 16, 16), 1.0, 5.0)


def config1() -> Case:
    """BASELINE config 1: 4 views 256^2, C=32, Bp + 2 U&F steps."""
    return _rig_case("config1", q.config1(), q.RigSpec(2, 2, 0.1, 256, 256, 256.0),
                     q.Camera.make(256, 256, 128, 128, 256, 256), 1.0, 20.0)


def config2(div: int = 1, views_rig=(2, 4), baseline=0.1) -> Case:
    """BASELINE config 2 (div=1): 8 views, full_scale_config, encoder
    576x960, render 1080x1920, target at the rig centroid, near 0.5 far 100.
    div > 1 gives the same schedule with every extent / div (the bounded
    CPU-baseline sample)."""
    rows, cols = views_rig
    cfg = q.full_scale_config() if div == 1 else q.scaled_full_config(div)
    cfg = replace(cfg, views=rows * cols)
    Hr, Wr = 1080 // div, 1920 // div
    He, We = 576 // div, 960 // div
    rcams, tgt = q.rig_cameras(q.RigSpec(rows, cols, baseline, Wr, Hr, 1080.0 / div))
    target = q.Frustum(tgt, 0.5, 100.0)
    ecams = [c.scaled(We, He) for c in rcams]
    eimgs = q.scene_images(21, 3, target, ecams)
    rimgs = q.scene_images(21, 3, target, rcams)
    return Case(f"config2_div{div}_m{rows * cols}", cfg, eimgs, ecams, rimgs, rcams, target)
