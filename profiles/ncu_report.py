"""One-screen report of an ncu --set full capture: the headline throughputs
(profiles/ncu_brief.py's fields), the warp-stall reasons, and the source
lines with the most stall samples (-lineinfo builds).

  python profiles/ncu_report.py gpurun_out/full_<kernel>_<skip>.ncu-rep > profiles/r2/ncu_<name>.txt
"""
import collections
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "No Eligible", "Executed Instructions", "Grid Size", "Block Size", "L1/TEX Hit Rate",
        "L2 Hit Rate"]


def run(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, top=15):
    rows = list(csv.reader(io.StringIO(run(rep, "--page", "details", "--csv"))))
    h = rows[0]
    print(rows[1][h.index("Kernel Name")][:110])
    seen = set()
    for r in rows[1:]:
        name, unit, val = r[h.index("Metric Name")], r[h.index("Metric Unit")], r[h.index("Metric Value")]
        if name in WANT and name not in seen:
            seen.add(name)
            print(f"  {name:40s} {val:>16s} {unit}")
    raw = list(csv.reader(io.StringIO(run(rep, "--page", "raw", "--csv"))))
    d = dict(zip(raw[0], raw[2] if len(raw) > 2 else raw[1]))
    st = []
    for k, v in d.items():
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                st.append((float(v.replace(",", "")), k.split("stalled_")[-1]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    print("  warp-stall samples by reason:")
    for x, k in sorted(st, reverse=True)[:8]:
        print(f"    {x / tot * 100:5.1f}%  {k}")
    src = list(csv.reader(io.StringIO(run(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    cur_file = cur_line = None
    agg = collections.Counter()
    seen = set()
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or len(r) < 5:
            continue
        if r[0]:
            cur_line = (cur_file, r[0], r[1].strip()[:90])
        if r[2] and (r[2], cur_line) not in seen:
            seen.add((r[2], cur_line))
            try:
                agg[cur_line] += float(r[4] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1.0
    print(f"  top source lines by warp-stall samples ({int(tot)} samples):")
    for k, v in agg.most_common(top):
        print(f"    {v / tot * 100:5.1f}%  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1])
