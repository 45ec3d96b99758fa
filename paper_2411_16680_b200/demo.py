"""forward-demo on the B200 path (the reference CLI's run_forward_demo,
tools/main.cpp:511-611): one synthetic scene through forward + render_target,
the outputs written to a directory, and the paper's per-view cost
decomposition T = T_V + M * T_image (the reference fits it to
scalar-op counts at M = 2, 4, 8, main.cpp:577-604) fitted to MEASURED device
time per frame on this GPU, at M = 4, 8, 16 (the view counts the kernels are
specialised for).

    python -m paper_2411_16680_b200.demo --out /tmp/demo            # config 2
    python -m paper_2411_16680_b200.demo --workload config1 --weights store.qntc

Outputs: target.npy [Ho,Wo,3] f32, ldm.qntc (the activated LDM: depth,
density, blend, blend_logits as f32 QNTC entries, io.cpp:100-124 layout),
weights.qntc (the bound parameter store, named by NetParams member path),
timings.json (per-M device ms/frame, T_V, T_image, the residual of the third
point, and the launch count per frame). Scene bundles / PFM are out of scope
(DESIGN.md §7): the scene is the synthetic workload of `--workload`.
"""
from __future__ import annotations

import argparse
import json
import os
from dataclasses import replace

import numpy as np

from . import qntc
from . import workloads as wl
from .config import model_config_from_json
from .lvs import Model, plan_forward

WORKLOADS = {"config1": lambda: wl.config1(), "config2": lambda: wl.config2(),
             "config2_div4": lambda: wl.config2(div=4), "nano": lambda: wl.nano()}
# The per-view sweep needs up to 16 views: config 2's workloads sweep the
# first M cameras of config 3's 4 x 4 rig (same schedule, same extents). The
# view-count-specialised kernels cover M = 4, 8, 16; other M run the generic
# SIMT fallbacks and are not representative.
SWEEP_CASES = {"config2": lambda: wl.config3(), "config2_div4": lambda: wl.config3(div=4)}


def _device_ms(cfg, case, views: int, frames: int, weights: bytes) -> tuple:
    """Median device ms per frame of forward+render at `views` input views
    (the first `views` cameras of the case), inputs resident, and the launch
    count of one frame."""
    import torch
    dev = torch.device("cuda", 0)
    c = replace(cfg, views=views)
    m = Model(c, device=0)
    m.load_weights_qntc(weights)  # parameter shapes never depend on M
    enc = torch.from_numpy(np.ascontiguousarray(case.enc_images[:views])).to(dev)
    ren = torch.from_numpy(np.ascontiguousarray(case.ren_images[:views])).to(dev)
    plan = plan_forward(c, enc.shape[1], enc.shape[2])
    out = torch.empty((plan.out_height, plan.out_width, 3), device=dev)
    st = torch.cuda.Stream(dev)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)  # 256 MB > L2
    args = (enc, case.enc_cams[:views], ren, case.ren_cams[:views], case.target, out)
    for _ in range(3):
        m.forward_render_device(*args, stream=st)
    launches = m.last_launch_count()
    times = []
    with torch.cuda.stream(st):
        for _ in range(frames):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            m.forward_render_device(*args, stream=st)
            e1.record(st)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    m.close()
    return float(np.median(times)), int(launches)


def run(workload: str, out_dir: str, seed: int = 3, weights_path: str | None = None,
        config_path: str | None = None, sweep=(2, 4, 8, 16), frames: int = 10) -> dict:
    case = WORKLOADS[workload]()
    cfg = case.cfg
    if config_path:
        with open(config_path) as f:
            cfg = model_config_from_json(f.read())
        if cfg.views != case.cfg.views:
            raise ValueError(f"forward-demo: the config expects {cfg.views} views but the "
                             f"workload has {case.cfg.views}")
    os.makedirs(out_dir, exist_ok=True)
    if weights_path:
        with open(weights_path, "rb") as f:
            weights = f.read()
    else:
        weights = qntc.pack_param_store(cfg, seed)
    with open(os.path.join(out_dir, "weights.qntc"), "wb") as f:
        f.write(weights)

    m = Model(cfg, device=0)
    m.load_weights_qntc(weights)
    ldm = m.forward(case.enc_images, case.enc_cams, case.target)
    rgb = m.render_target(case.ren_images, case.ren_cams)
    np.save(os.path.join(out_dir, "target.npy"), rgb)
    with open(os.path.join(out_dir, "ldm.qntc"), "wb") as f:
        f.write(qntc.pack_tensors([("depth", ldm.depth), ("density", ldm.density),
                                   ("blend", ldm.blend), ("blend_logits", ldm.blend_logits)]))
    m.close()

    pts = {}
    scase = SWEEP_CASES.get(workload, lambda: case)()
    for v in sweep:
        if v > scase.enc_images.shape[0]:
            continue
        ms, launches = _device_ms(cfg, scase, v, frames, weights)
        pts[v] = {"ms_per_frame": ms, "launches": launches}
    res = {"workload": workload, "views": cfg.views, "out_hw": list(rgb.shape[:2]),
           "sweep_case": scase.name, "per_view_ms": pts}
    ms_ = sorted(pts)
    if len(ms_) >= 2:
        (m0, m1) = ms_[:2]
        t_image = (pts[m1]["ms_per_frame"] - pts[m0]["ms_per_frame"]) / (m1 - m0)
        t_volume = pts[m0]["ms_per_frame"] - m0 * t_image
        res.update(t_volume_ms=t_volume, t_image_ms=t_image)
        if len(ms_) >= 3:
            m2 = ms_[2]
            res["residual_ms"] = pts[m2]["ms_per_frame"] - (t_volume + m2 * t_image)
            xs = np.array(ms_, float)
            ys = np.array([pts[k]["ms_per_frame"] for k in ms_])
            slope, icpt = np.polyfit(xs, ys, 1)
            res.update(lsq_t_volume_ms=float(icpt), lsq_t_image_ms=float(slope))
    with open(os.path.join(out_dir, "timings.json"), "w") as f:
        json.dump(res, f, indent=2)
    return res


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--workload", default="config2", choices=sorted(WORKLOADS))
    ap.add_argument("--config", default=None, help="ModelConfig JSON (io.cpp:571-633)")
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--weights", default=None, help="QNTC parameter store")
    ap.add_argument("--out", required=True)
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--sweep", default="2,4,8,16")
    a = ap.parse_args(argv)
    res = run(a.workload, a.out, a.seed, a.weights, a.config,
              tuple(int(x) for x in a.sweep.split(",") if x), a.frames)
    for v, p in res["per_view_ms"].items():
        print(f"views {v}: {p['ms_per_frame']:.3f} ms/frame ({p['launches']} launches)")
    if "t_image_ms" in res:
        print(f"decomposition: {res['t_volume_ms']:.3f} + views x {res['t_image_ms']:.3f} ms "
              f"(residual {res.get('residual_ms', 0.0):.3f} ms)")
    print(f"wrote forward-demo outputs to {a.out}")


if __name__ == "__main__":
    main()
