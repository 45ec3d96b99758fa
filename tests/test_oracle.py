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


def test_flip_attribution_metrics(oracle):
    """tests/parity_util.py on the oracle's own nano frame: identical depth
    gives no flips and zero error; a depth perturbation large enough to move
    footprints across a view edge is reported as flip pixels."""
    import numpy as np
    from cases import nano
    from parity_util import flip_mask, frame_metrics, gate
    case = nano()
    want = oracle.forward_render(case.cfg, case.enc_images, case.enc_cams, case.ren_images,
                                 case.ren_cams, case.target, case.flat(), outputs=("rgb", "depth"))
    m = frame_metrics(oracle, case, want["rgb"], want["depth"], want)
    assert m["rgb_max_abs"] == 0.0 and m["flip_px"] == 0 and gate(m)
    d2 = want["depth"] * np.float32(1.3)
    fl = flip_mask(oracle, case.target, case.ren_cams, want["depth"], d2)
    assert fl.shape == want["depth"].shape[1:] and fl.any()


@pytest.mark.parametrize("heads,M,zero", [(1, 4, False), (2, 8, False), (4, 16, False),
                                          (2, 8, True)])
def test_attend_residual_stage_matches_reference(oracle, reference, heads, M, zero):
    """The oracle's attend_residual export (per-stage parity input, SURVEY.md
    §7.2 step 1) is bit-identical to the reference's (attention.hpp:248-252)."""
    import numpy as np
    rng = np.random.default_rng(7 + heads + M)
    P_, C = 777, 32
    V = rng.standard_normal((P_, C)).astype(np.float32)
    D = rng.standard_normal((P_, M, C)).astype(np.float32)
    wq = (rng.standard_normal((heads, C, C)) / np.sqrt(C)).astype(np.float32)
    wo = (0.1 * rng.standard_normal((heads * C, C)) / np.sqrt(heads * C)).astype(np.float32)
    g = (1 + 0.1 * rng.standard_normal(C)).astype(np.float32)
    a = oracle.attend_residual(V, D, wq, wo, g, zero)
    b = reference.attend_residual(V, D, wq, wo, g, zero)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert not np.array_equal(a, V)


def test_render_to_view_stage_matches_reference(oracle, reference):
    """The oracle's render_to_input_view export (ldm.hpp:223-244, the splat
    into one input view) is bit-identical to the reference's, on the
    oracle's own config-1 final volume."""
    import numpy as np
    from cases import config1
    from paper_2411_16680_b200.qntc import param_names
    case = config1()
    V = oracle.forward_render(case.cfg, case.enc_images, case.enc_cams, None, None, case.target,
                              case.flat(), outputs=("volume",))["volume"]
    w = dict(zip(param_names(case.cfg), case.store()))
    cam = case.enc_cams[1].scaled(48, 40)
    a, bad = oracle.render_to_view(case.target, V, w["heads.w_appear"], w["heads.w_sigma"],
                                   w["heads.w_depth"], cam)
    b = reference.render_to_view(case.target, V, w["heads.w_appear"], w["heads.w_sigma"],
                                 w["heads.w_depth"], cam)
    assert not bad and a.shape == (40, 48, 33)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert a[..., -1].max() > 0.5
