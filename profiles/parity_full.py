"""Full-scale parity sweep over BASELINE configs 2-5 (1080p, every frame /
target) against the oracle, with validity-flip attribution
(tests/parity_util.py). One JSON line per frame to stdout and to --out.

  python profiles/parity_full.py --cases c4 c5 --out gpurun_out/parity_full.jsonl
  cases: c2 (config 2), c3 (config 3), c4 (30 video frames), c5 (8 targets),
         c4:T / c5:K for a single frame / target
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)


def expand(names):
    from paper_2411_16680_b200 import workloads as wl
    grid = wl.config5_targets()
    for n in names:
        if n == "c2":
            yield lambda: wl.config2(div=1)
        elif n == "c3":
            yield lambda: wl.config3(div=1)
        elif n == "c4":
            for t in range(30):
                yield (lambda t=t: wl.config4_frame(t, div=1))
        elif n.startswith("c4:"):
            t = int(n[3:])
            yield (lambda t=t: wl.config4_frame(t, div=1))
        elif n == "c5" or n.startswith("c5:"):
            ks = range(8) if n == "c5" else [int(n[3:])]
            for k in ks:
                def mk(k=k):
                    c = wl.config2(div=1, target_center=grid[k])
                    c.name = f"config5_target{k}"
                    return c
                yield mk
        else:
            raise SystemExit(f"unknown case {n}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="+", default=["c4", "c5"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--self-runs", type=int, default=0,
                    help="for each frame over the plain gate, re-run the oracle this many times "
                         "with its inputs moved by one ulp (tests/parity_util.self_sensitivity)")
    a = ap.parse_args()
    import paper_2411_16680_b200 as q
    from bindings import Oracle
    from parity_util import RGB_MAX_ABS, full_frame_check, self_sensitivity
    oracle = Oracle()
    model = None
    fails = 0
    out = open(a.out, "a") if a.out else None
    for mk in expand(a.cases):
        case = mk()
        t0 = time.time()
        if model is None or model.cfg.views != case.cfg.views:
            model = q.Model(case.cfg, device=0)
            model.load_weights(case.store())
        rgb = model.forward_render(case.enc_images, case.enc_cams, case.ren_images, case.ren_cams,
                                   case.target)
        depth = model.forward(case.enc_images, case.enc_cams, case.target).depth
        t1 = time.time()
        m = full_frame_check(oracle, case, rgb, depth)
        t2 = time.time()
        m["plain_gate"] = m["rgb_max_abs"] <= RGB_MAX_ABS
        m["gpu_s"], m["oracle_s"] = round(t1 - t0, 2), round(t2 - t1, 2)
        # keep only the events next to pixels over the gate
        m["internal_events"] = m["internal_events"][:8] if m["px_gt_1e-3_internal"] else []
        if not m["plain_gate"] and a.self_runs:
            want = oracle.forward_render(case.cfg, case.enc_images, case.enc_cams, case.ren_images,
                                         case.ren_cams, case.target, case.flat(),
                                         outputs=("rgb", "depth"))
            runs = []
            for k in range(a.self_runs):
                spx, sfl, _ = self_sensitivity(oracle, case, want, seed=1000 + 17 * k)
                runs.append({"max_abs": float(spx.max()), "px_gt_1e-3": int((spx > RGB_MAX_ABS).sum()),
                             "px_gt_1e-4": int((spx > 1e-4).sum()), "flip_px": int(sfl.sum())})
            m["self_runs"] = runs
        fails += not m["pass"]
        line = json.dumps(m)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()
    print(f"parity_full: {fails} failing frame(s) (attributed gate)")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
