"""DRAM traffic of one frame from an ncu launch list with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(--csv, --clock-control none) of `bench.py --steps 1 --warmup 3 --no-e2e
--no-cpu-baseline`: the launches of the last frame (from its encoder stem to
the end, torch's own kernels dropped), summed per kernel family.

  python profiles/traffic_summary.py gpurun_out/traffic.csv > profiles/r2/traffic.json

bench.py reads profiles/r2/traffic.json for the conv roofline's `traffic`
and the frame-level DRAM GB/s. Under ncu every launch is serialised and
replayed, so bytes are per launch in isolation (no inter-kernel L2 reuse).
"""
import collections
import csv
import json
import re
import sys


def family(name):
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"lvsg::(<unnamed>::)?", "", n).replace("void ", "")
    base = re.sub(r"<.*", "", n)
    if base.startswith("conv3x3") and "weights" not in base:
        return "conv3x3" if "stem" not in base else "conv3x3_stem"
    return base


def main():
    path = sys.argv[1]
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("ID"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    seq = list(launches.values())
    starts = [i for i, d in enumerate(seq) if "stem3x2" in d["name"] or "conv3x3_stem" in d["name"]]
    frame = [d for d in seq[starts[-1]:] if "lvsg" in d["name"]]
    fam = collections.OrderedDict()
    tot_b = tot_t = 0.0
    for d in frame:
        f = family(d["name"])
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        t = d.get("gpu__time_duration.sum", 0.0)
        e = fam.setdefault(f, {"launches": 0, "dram_bytes": 0.0, "ns": 0.0})
        e["launches"] += 1
        e["dram_bytes"] += b
        e["ns"] += t
        tot_b += b
        tot_t += t
    out = {"source": f"{path} (ncu, last frame, {len(frame)} lvsg launches)",
           "frame_dram_bytes": tot_b, "frame_serialised_ns": tot_t,
           "families": {k: dict(v, gbs=v["dram_bytes"] / max(v["ns"], 1.0)) for k, v in fam.items()}}
    if "conv3x3" in fam:
        c = fam["conv3x3"]
        out["conv3x3"] = {"launches": c["launches"], "dram_bytes_per_frame": c["dram_bytes"],
                          "serialised_ns": c["ns"], "source": out["source"]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
