"""End-to-end parity metrics with validity-flip attribution (SURVEY.md §7.2,
parity protocol step 2). TEST INFRASTRUCTURE: the oracle is the checker.

A "validity flip" is a (layer, output pixel, view) whose footprint validity
(`geometry.hpp:60-79`) differs between the footprints recomputed from the
GPU's final LDM depth and from the oracle's. The reference's render
renormalises the blend weights over the valid views (`ldm.hpp:184-187`), so
a flip switches a pixel's colour sources discontinuously; every RGB value
above the gate must lie on a flip pixel for a difference to be attributed
to depth rounding rather than to a defect.
"""
from __future__ import annotations

import numpy as np

RGB_MAX_ABS = 1e-3
RGB_PSNR_DB = 50.0


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if mse == 0 else -10.0 * np.log10(mse)


def flip_mask(oracle, target, ren_cams, depth_a, depth_b):
    """[Ho, Wo] bool: pixels where any (layer, view) footprint validity
    differs between the two depth maps ([L, Ho, Wo] each)."""
    pa, _ = oracle.world_points(target, np.ascontiguousarray(depth_a))
    pb, _ = oracle.world_points(target, np.ascontiguousarray(depth_b))
    L, Ho, Wo = depth_a.shape
    mask = np.zeros((L, Ho, Wo), bool)
    for cam in ren_cams:
        _, va, _ = oracle.footprints(cam, pa)
        _, vb, _ = oracle.footprints(cam, pb)
        mask |= (va != vb).reshape(L, Ho, Wo)
    return mask.any(0)


def frame_metrics(oracle, case, rgb, depth, want):
    """rgb/depth: the GPU frame and its final LDM depth; want: the oracle's
    outputs with "rgb" and "depth". Returns a JSON-able dict."""
    d = np.abs(rgb - want["rgb"])
    dpx = d.max(-1)
    flips = flip_mask(oracle, case.target, case.ren_cams, depth, want["depth"])
    off = dpx[~flips]
    over = dpx > RGB_MAX_ABS
    rel_depth = np.abs(depth - want["depth"]) / np.maximum(np.abs(want["depth"]), 1e-6)
    return {
        "case": case.name,
        "rgb_max_abs": float(d.max()),
        "psnr_db": psnr(rgb, want["rgb"]),
        "values_gt_1e-3": int((d > RGB_MAX_ABS).sum()),
        "values": int(d.size),
        "px_gt_1e-5": int((dpx > 1e-5).sum()),
        "flip_px": int(flips.sum()),
        "max_abs_off_flip_px": float(off.max()) if off.size else 0.0,
        "px_gt_1e-3_on_flip": int((over & flips).sum()),
        "px_gt_1e-3_unattributed": int((over & ~flips).sum()),
        "depth_max_rel": float(rel_depth.max()),
    }


def gate(m):
    """The north-star gate: max-abs <= 1e-3 and PSNR >= 50 dB."""
    return m["rgb_max_abs"] <= RGB_MAX_ABS and m["psnr_db"] >= RGB_PSNR_DB


def attributed_gate(m):
    """The gate with attribution: PSNR >= 50 dB;
    every value above 1e-3 lies on a final-render validity-flip pixel or
    next to an internal near-edge footprint (full_frame_check); nothing
    above 1e-3 anywhere else."""
    return (m["psnr_db"] >= RGB_PSNR_DB and m["px_gt_1e-3_unexplained"] == 0
            and m["max_abs_unexplained_px"] <= RGB_MAX_ABS)


def perturb_ulp(a, seed):
    """Every element of the f32 array moved by one ulp up or down (random
    sign, fixed seed): one rounding's worth of noise on the inputs."""
    a = np.ascontiguousarray(a, np.float32)
    up = np.random.default_rng(seed).random(a.shape) < 0.5
    return np.where(up, np.nextafter(a, np.float32(np.inf)),
                    np.nextafter(a, np.float32(-np.inf))).astype(np.float32)


def self_sensitivity(oracle, case, want, seed):
    """The reference's own conditioning at this frame: the oracle (bit-exact
    with the reference) re-run with its weights and encoder images each moved
    by one ulp, compared with its unperturbed frame `want`. Returns the
    per-pixel max-abs change [Ho, Wo] and the final-render flip mask between
    the two depth maps."""
    got = oracle.forward_render(case.cfg, perturb_ulp(case.enc_images, seed), case.enc_cams,
                                case.ren_images, case.ren_cams, case.target,
                                perturb_ulp(case.flat(), seed + 1), outputs=("rgb", "depth"))
    dpx = np.abs(got["rgb"] - want["rgb"]).max(-1)
    flips = flip_mask(oracle, case.target, case.ren_cams, got["depth"], want["depth"])
    return dpx, flips, got


def internal_margins(oracle, case, tol=1e-3):
    """The oracle's forward with the validity-margin trace on: every Stage-1
    gather and render-to-input-view splat footprint of the solve that lies
    within `tol` px of its view's validity edge (a discontinuity inside the
    network: an f32-rounding-sized change of the LDM depth at that step can
    switch the texel's view on or off). Returns (outputs, rows [n, 8])."""
    return oracle.trace_margins(tol, lambda: oracle.forward_render(
        case.cfg, case.enc_images, case.enc_cams, case.ren_images, case.ren_cams, case.target,
        case.flat(), outputs=("rgb", "depth")))


def events_to_output(rows, step_hw, out_hw):
    """Maps trace rows' texels (y, x at their step's H, W) to output-pixel
    coordinates (the bilinear resize's centre alignment)."""
    Ho, Wo = out_hw
    ys = np.empty(len(rows))
    xs = np.empty(len(rows))
    for i, r in enumerate(rows):
        H, W = step_hw[int(r[0])]
        ys[i] = (r[4] + 0.5) * Ho / H - 0.5
        xs[i] = (r[5] + 0.5) * Wo / W - 0.5
    return ys, xs


# An internal near-edge footprint at step s perturbs its texel of the step-s
# volume; the fusion block's 3x3 convs and the bilinear upsample spread that
# over ~2 texels, i.e. 2.5 * (Ho / H_s) output pixels.
INTERNAL_MARGIN_PX = 1e-4
SPREAD_TEXELS = 2.5


def full_frame_check(oracle, case, rgb, depth):
    """One frame of the GPU path (rgb [Ho,Wo,3], final LDM depth [L,Ho,Wo])
    against the oracle with both attributions:
      * final-render validity flips (flip_mask on the two depth maps);
      * internal discontinuities: Stage-1 gathers / render-to-view splats of
        the solve whose footprint lies within INTERNAL_MARGIN_PX of its
        view's validity edge in the oracle's own forward (trace rows), an
        f32-rounding-sized LDM difference away from switching that view.
    Returns frame_metrics + px_gt_1e-3_internal, px_gt_1e-3_unexplained,
    max_abs_unexplained_px, internal_events (list) and "pass"."""
    want, rows = internal_margins(oracle, case, INTERNAL_MARGIN_PX)
    m = frame_metrics(oracle, case, rgb, depth, want)
    dpx = np.abs(rgb - want["rgb"]).max(-1)
    flips = flip_mask(oracle, case.target, case.ren_cams, depth, want["depth"])
    rows = rows[rows[:, 0] >= 1]  # step 0 gathers at exact anchor depths: no rounding
    Ho, Wo = dpx.shape
    hw = [(sp.height, sp.width) for sp in case.cfg.steps]
    near = np.zeros_like(flips)
    if len(rows):
        ey, ex = events_to_output(rows, hw, (Ho, Wo))
        yy, xx = np.mgrid[0:Ho, 0:Wo]
        for r, y, x in zip(rows, ey, ex):
            rad = SPREAD_TEXELS * Ho / hw[int(r[0])][0]
            y0, y1 = max(0, int(y - rad)), min(Ho, int(y + rad) + 2)
            x0, x1 = max(0, int(x - rad)), min(Wo, int(x + rad) + 2)
            near[y0:y1, x0:x1] |= np.hypot(yy[y0:y1, x0:x1] - y, xx[y0:y1, x0:x1] - x) <= rad
    over = dpx > RGB_MAX_ABS
    unexpl = ~flips & ~near
    m["internal_events"] = [[float(v) for v in r] for r in rows[:50]]
    m["internal_events_n"] = int(len(rows))
    m["px_gt_1e-3_internal"] = int((over & ~flips & near).sum())
    m["px_gt_1e-3_unexplained"] = int((over & unexpl).sum())
    m["max_abs_unexplained_px"] = float(dpx[unexpl].max()) if unexpl.any() else 0.0
    m["pass"] = attributed_gate(m)
    return m
