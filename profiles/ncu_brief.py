"""One-screen summary of an ncu --set full report: duration, throughputs,
issue, occupancy, the warp-stall breakdown and the top source lines."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "No Eligible", "Executed Instructions", "Grid Size", "Block Size", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Mem Pipes Busy"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    print(rows[1][h.index("Kernel Name")][:90])
    for r in rows[1:]:
        n = r[h.index("Metric Name")]
        if n in WANT:
            print(f"  {n:38s} {r[h.index('Metric Value')]:>14s} {r[h.index('Metric Unit')]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        names, vals = rr[0], rr[2]
        st = [(n, v) for n, v in zip(names, vals)
              if n.startswith("smsp__average_warp_latency_issue_stalled_") and n.endswith(".ratio")]
        tot = 0.0
        parsed = []
        for n, v in st:
            try:
                parsed.append((float(v), n.replace("smsp__average_warp_latency_issue_stalled_", "")
                               .replace(".ratio", "")))
            except ValueError:
                pass
        parsed.sort(reverse=True)
        print("  stalls (cycles per issued instruction):",
              ", ".join(f"{n} {v:.2f}" for v, n in parsed[:8]))


if __name__ == "__main__":
    for r in sys.argv[1:]:
        main(r)
