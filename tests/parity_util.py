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
    """The north-star gate plus attribution: max-abs and PSNR within the
    tolerance, and nothing above it off the flip pixels."""
    return (m["rgb_max_abs"] <= RGB_MAX_ABS and m["psnr_db"] >= RGB_PSNR_DB
            and m["px_gt_1e-3_unattributed"] == 0)


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
