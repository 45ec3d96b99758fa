"""Host-side logic of the native library (no GPU): config grammar and
validation (network.cpp:8-103), plan_forward (network.cpp:105-151), the
build_params weight layout and bit-exact init RNG, the synthetic scene
generator, and the C ABI surface."""
import ctypes
import os
import re
from dataclasses import replace

import numpy as np
import pytest

import paper_2411_16680_b200 as q
from paper_2411_16680_b200 import capi
from bindings import fnv1a64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "lvsg.h")).read()
    declared = set(re.findall(r"\b(lvsg_[a-z_0-9]+)\s*\(", hdr))
    lib = capi.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(capi.SYMBOLS)


def test_create_without_gpu_fails_cleanly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(q.DeviceError):
        q.Model(q.nano_config())


def test_production_plan_matches_reference_golden():
    g = np.load(os.path.join(GOLDEN, "plan.npz"))
    p = q.plan_forward(q.full_scale_config(), 576, 960)
    assert [list(x) for x in g["pyramid"]] == [list(x) for x in p.pyramid]
    got = [[s.in_layers, s.layers, s.in_height, s.in_width, s.height, s.width, int(s.doubled),
            s.level, s.feat_h, s.feat_w, s.render_h, s.render_w, s.collapse_count] for s in p.steps]
    assert got == g["steps"].tolist()
    assert (p.out_height, p.out_width) == tuple(g["out"])


def test_plan_matches_live_reference(reference):
    for cfg, (h, w) in [(q.nano_config(), (64, 64)), (q.config1(), (256, 256)),
                        (q.scaled_full_config(4), (144, 240)), (q.micro_config(), (16, 16))]:
        p = q.plan_forward(cfg, h, w)
        r = reference.plan_forward(cfg, h, w)
        assert p.out_height == r.out_height and p.out_width == r.out_width
        for s, rs in zip(p.steps, list(r.steps)[:r.num_steps]):
            assert (s.render_h, s.render_w, s.feat_h, s.feat_w, s.doubled) == \
                (rs.render_h, rs.render_w, rs.feat_h, rs.feat_w, bool(rs.doubled))


def _broken(mut):
    cfg = q.nano_config()
    cfg = replace(cfg, steps=[replace(s) for s in cfg.steps])
    mut(cfg)
    with pytest.raises(q.DimError):
        q.validate_config(cfg)


def test_validation_rejects_bad_configs():
    """test_network.cpp:60-110: grammar and chaining rules."""
    q.validate_config(q.nano_config())
    q.validate_config(q.full_scale_config())

    def setb(i, b):
        return lambda c: setattr(c.steps[i], "blocks", b)
    for mut in [setb(0, "U,A2,C"), setb(1, "Bp,A2,C"), setb(0, "Lc,Bp,A2"), setb(1, "U,C"),
                setb(1, "U"), setb(1, "U,A2,Lc"), setb(1, "U,A0"), setb(1, "U,Ax"),
                setb(1, "X,A2"), setb(1, "U,A2,"), setb(1, ""),
                lambda c: setattr(c.steps[3], "in_layers", 4),
                lambda c: (setattr(c.steps[2], "height", 24), setattr(c.steps[2], "width", 24)),
                lambda c: setattr(c.steps[1], "pyramid_level", 3),
                lambda c: setattr(c.steps[0], "in_layers", 16),
                lambda c: setattr(c, "upsample", 0.5),
                lambda c: (setattr(c, "near", 2.0), setattr(c, "far", 1.0)),
                lambda c: setattr(c, "views", 0), lambda c: setattr(c, "channels", 0),
                lambda c: setattr(c, "steps", [])]:
        _broken(mut)
    # whitespace around tokens is accepted (network.cpp:18-19)
    cfg = q.nano_config()
    cfg.steps[1].blocks = " U , A2 ,\tC,C"
    q.validate_config(cfg)


def test_plan_rejects_unhalvable_images():
    with pytest.raises(q.DimError):
        q.plan_forward(q.nano_config(), 63, 64)
    with pytest.raises(q.DimError):
        q.plan_forward(q.nano_config(), 64, 62)
    with pytest.raises(q.DimError):  # the 1080p trap of SURVEY.md §0
        q.plan_forward(q.full_scale_config(), 1080, 1920)
    cfg = q.micro_config()
    cfg.pyramid_levels = 1
    cfg.steps[0].pyramid_level = 0
    with pytest.raises(q.DimError):  # doubling step without a coarser level
        q.plan_forward(cfg, 16, 16)


def test_param_layout_counts():
    """312 tensors / 1,095,424 params at full scale, 119 at
    nano; shapes never depend on M (test_network.cpp:265-271)."""
    shapes = q.param_shapes(q.full_scale_config())
    assert len(shapes) == 312
    assert sum(int(np.prod(s)) for s in shapes) == 1095424
    assert shapes[44] == (32, 64, 3, 3) and shapes[250] == (64, 64)
    assert len(q.param_shapes(q.nano_config())) == 119
    assert q.param_shapes(q.full_scale_config().with_views(16)) == shapes


def test_init_param_store_bit_exact(reference):
    for cfg in (q.nano_config(), q.full_scale_config(), replace(q.nano_config(), direct_rgb=True)):
        a = q.init_param_store(cfg, 3, flat=True)
        b, _, _ = reference.init_param_store(cfg, 3)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_scene_generator_bit_exact(reference):
    cams, tgt = q.rig_cameras(q.RigSpec(2, 4, 0.1, 192, 108, 108.0))
    rc, rt = reference.rig(2, 4, 0.1, 192, 108, 108.0)
    for a, b in zip(cams, rc):
        assert np.array_equal(a.cam_from_world.reshape(-1), np.array(list(b.cam_from_world)))
    fr = q.Frustum(tgt, 0.5, 100.0)
    a = q.scene_images(21, 3, fr, cams)
    b = reference.scene_images(21, 3, fr, cams)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert a.min() > 0.0 and a.max() < 1.0
    # config 4's moving content: planes but the backdrop shifted along x
    a = q.scene_images(21, 3, fr, cams, shift_x=0.07)
    b = reference.scene_images(21, 3, fr, cams, shift_x=0.07)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert not np.array_equal(a, q.scene_images(21, 3, fr, cams))


def test_camera_helpers():
    c = q.Camera.make(100, 80, 50, 40, 100, 80)
    s = c.scaled(50, 20)
    assert (s.fx, s.fy, s.cx, s.cy, s.width, s.height) == (50, 20, 25, 10, 50, 20)
    with pytest.raises(q.DimError):
        q.Camera.make(-1, 1, 0, 0, 4, 4)
    bad = np.eye(4)
    bad[0, 0] = 2
    with pytest.raises(q.DimError):
        q.Camera.make(1, 1, 0, 0, 4, 4, bad)
    with pytest.raises(q.DimError):
        q.Frustum(c, 2.0, 1.0).validate()
