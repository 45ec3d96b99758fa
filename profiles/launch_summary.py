"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total device time, launch count and share. With --last-frame,
only launches after the last L2-flush fill kernel (bench.py flushes before
every timed frame) are counted, i.e. exactly one timed frame."""
import collections
import csv
import sys


def main(path, last_frame=False):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    body = [r for r in rows[hdr + 1:] if len(r) > vi]
    if last_frame:
        flush = [i for i, r in enumerate(body) if "FillFunctor" in r[ki]]
        if flush:
            body = body[flush[-1] + 1:]
    agg = collections.defaultdict(lambda: [0.0, 0])
    tot = 0.0
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
    for r in body:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("lvsg::", "")
        name = name.replace("<unnamed>::", "")
        agg[name][0] += v
        agg[name][1] += 1
        tot += v
    print(f"{'ms':>9} {'n':>5} {'share':>6}  kernel")
    for k, (v, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{v:9.3f} {n:5d} {100 * v / tot:5.1f}%  {k[:100]}")
    print(f"{tot:9.3f} total (cold-cache, serialised replay)")


if __name__ == "__main__":
    main(sys.argv[1], "--last-frame" in sys.argv)
