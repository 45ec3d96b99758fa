"""Calibrates bench.py's bounded CPU sample: one FULL config-2 frame of the
reference (oracle/_ref, single-threaded, forward + render_target) timed on
this host, next to the 1/4-extent sample bench.py extrapolates from.

  python profiles/ref_fullframe.py --out gpurun_out/ref_fullframe.json

Records seconds (forward / render / wall), peak RSS, CPU model and core count.
TEST / MEASUREMENT INFRASTRUCTURE: runs the reference only.
"""
import argparse
import json
import os
import resource
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run(div):
    """Child process: one reference frame at 1/div extents; prints JSON."""
    from bindings import Reference
    from paper_2411_16680_b200.workloads import config2
    import numpy as np
    c = config2(div=div)
    w = c.flat()
    r = Reference()
    t0 = time.perf_counter()
    out = r.forward_render(c.cfg, c.enc_images, c.enc_cams, c.ren_images, c.ren_cams, c.target, w,
                           outputs=("rgb",))
    wall = time.perf_counter() - t0
    rgb = out["rgb"]
    print(json.dumps({"div": div, "wall_s": wall, "fraction_of_frame": 1.0 / (div * div),
                      "rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
                      "rgb_mean": float(np.mean(rgb))}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--child", type=int, default=0)
    ap.add_argument("--divs", type=int, nargs="+", default=[4, 1])
    a = ap.parse_args()
    if a.child:
        run(a.child)
        return
    res = {"cpu_model": cpu_model(), "host_cores": os.cpu_count(), "threads_used": 1,
           "kind": "reference", "runs": []}
    for d in a.divs:
        p = subprocess.run([sys.executable, __file__, "--child", str(d)], capture_output=True,
                           text=True)
        line = [x for x in p.stdout.splitlines() if x.startswith("{")]
        res["runs"].append(json.loads(line[-1]) if line else {"div": d, "error": p.stderr[-500:]})
        print(json.dumps(res["runs"][-1]), flush=True)
    by = {r["div"]: r for r in res["runs"] if "wall_s" in r}
    if 1 in by and 4 in by:
        full, samp = by[1]["wall_s"], by[4]["wall_s"]
        res["full_frame_s"] = full
        res["sample_extrapolated_frame_s"] = samp * 16
        res["full_over_extrapolated"] = full / (samp * 16)
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
