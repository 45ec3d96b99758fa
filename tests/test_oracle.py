"""The oracle (oracle/lvs_oracle.c, a C restatement) pinned against the
reference itself: bit-exact against the committed golden fixtures made by the
reference build (tests/golden/make_golden.py) and, where oracle/_ref is
built, against the live reference on more cases. CPU only."""
import os
import subprocess

import numpy as np
import pytest

import paper_2411_16680_b200 as q
from bindings import REF_UNIT, fnv1a64
from cases import config1, micro, nano, nano_two_res

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
OUTS = ("rgb", "depth", "density", "blend", "blend_logits", "volume")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def test_inputs_match_golden():
    g = np.load(os.path.join(GOLDEN, "nano.npz"))
    c = nano()
    assert fnv1a64(c.flat()) == str(g["weights_fnv"])
    assert fnv1a64(c.enc_images) == str(g["images_fnv"])


def test_oracle_nano_bit_exact_vs_golden(oracle):
    g = np.load(os.path.join(GOLDEN, "nano.npz"))
    c = nano()
    r = oracle.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target,
                              c.flat(), outputs=OUTS)
    for k in OUTS:
        assert np.array_equal(bits(r[k]), bits(g[k])), k


def test_oracle_config1_bit_exact_vs_golden(oracle):
    g = np.load(os.path.join(GOLDEN, "config1.npz"))
    c = config1()
    assert fnv1a64(c.flat()) == str(g["weights_fnv"])
    r = oracle.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target,
                              c.flat())
    assert np.array_equal(bits(r["rgb"]), bits(g["rgb"]))
    assert fnv1a64(r["rgb"]) == str(g["rgb_fnv"])


def test_oracle_thread_count_does_not_change_bits(oracle):
    c = nano()
    a = oracle.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target,
                              c.flat())["rgb"]
    t = oracle.threads
    oracle.set_threads(1)
    try:
        b = oracle.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams,
                                  c.target, c.flat())["rgb"]
    finally:
        oracle.set_threads(t)
    assert np.array_equal(bits(a), bits(b))


def test_oracle_stages_vs_golden(oracle):
    g = np.load(os.path.join(GOLDEN, "stages.npz"))
    cv = g["cam"]
    cam = q.Camera(float(cv[16]), float(cv[17]), float(cv[18]), float(cv[19]), int(cv[20]),
                   int(cv[21]), cv[:16].reshape(4, 4).copy())
    from cases import config2
    c = config2(div=8)
    fr = q.Frustum(c.target.camera.scaled(80, 45), 0.5, 100.0)
    pts, bad = oracle.world_points(fr, g["depth"])
    assert not bad and np.array_equal(bits(pts), bits(g["points"]))
    taps, valid, fracs = oracle.footprints(cam, g["points"])
    assert np.array_equal(taps, g["taps"]) and np.array_equal(valid, g["valid"])
    assert np.array_equal(fracs, g["fracs"])
    assert fnv1a64(c.ren_images[1]) == str(g["image_fnv"])
    vals, mask = oracle.gather(cam, c.ren_images[1], g["points"])
    assert np.array_equal(bits(vals), bits(g["values"])) and np.array_equal(mask, g["mask"])
    assert 0 < valid.sum() < valid.size  # both valid and invalid footprints exercised


@pytest.mark.parametrize("make", [micro, nano_two_res, lambda: nano(ablate_render=True),
                                  lambda: nano(ablate_attention=True),
                                  lambda: nano(ablate_rays=True), lambda: nano(direct_rgb=True)],
                         ids=["micro", "two_res", "ablate_render", "ablate_attention",
                              "ablate_rays", "direct_rgb"])
def test_oracle_bit_exact_vs_live_reference(oracle, reference, make):
    c = make()
    # every ForwardResult field: the LDM, blend logits, volume, the final
    # step's deltas and, under direct_rgb, the decoded colour composite
    outs = OUTS + ("deltas",) + (("rgb_direct",) if c.cfg.direct_rgb else ())
    r = reference.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams,
                                 c.target, c.flat(), outputs=outs)
    o = oracle.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target,
                              c.flat(), outputs=outs)
    for k in outs:
        assert np.isfinite(r[k]).all(), k
        assert k not in ("deltas", "rgb_direct") or r[k].any(), k
        assert np.array_equal(bits(r[k]), bits(o[k])), k


def test_oracle_stage_functions_vs_live_reference(oracle, reference):
    c = nano()
    rng = np.random.default_rng(3)
    L, H, W, C, M = 3, 8, 8, 8, 4
    V = rng.standard_normal((L, H, W, C)).astype(np.float32)
    wd = rng.standard_normal((C, 1)).astype(np.float32) * 0.3
    ws = rng.standard_normal((C, 1)).astype(np.float32) * 0.3
    lg = rng.standard_normal((L, H, W, M)).astype(np.float32)
    a = reference.upsample_activate(c.target, V, wd, ws, lg, 20, 20)
    b = oracle.upsample_activate(c.target, V, wd, ws, lg, 20, 20)
    for x, y in zip(a, b):
        assert np.array_equal(bits(x), bits(y))
    rgb_r = reference.render_target(c.target, a[0], a[1], a[2], c.ren_images, c.ren_cams)
    rgb_o, bad = oracle.render_target(c.target, a[0], a[1], a[2], c.ren_images, c.ren_cams)
    assert not bad and np.array_equal(bits(rgb_r), bits(rgb_o))
    x = rng.standard_normal((5, 7, 9)).astype(np.float32)
    w = rng.standard_normal((4, 5, 3, 3)).astype(np.float32)
    bias = rng.standard_normal(4).astype(np.float32)
    y = oracle.conv3x3(x, w, bias)
    # independent naive check of the tap-skipping convention
    xp = np.pad(x.astype(np.float64), ((0, 0), (1, 1), (1, 1)))
    want = np.zeros((4, 7, 9))
    for co in range(4):
        want[co] = bias[co]
        for ci in range(5):
            for di in range(3):
                for dj in range(3):
                    want[co] += w[co, ci, di, dj] * xp[ci, di:di + 7, dj:dj + 9]
    assert np.abs(y - want).max() < 1e-4


def test_reference_unit_suite_passes(reference):
    """The reference's own 93-case doctest suite, built against the shims."""
    if not os.path.exists(REF_UNIT):
        pytest.skip("lvs_unit not built")
    r = subprocess.run([REF_UNIT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
