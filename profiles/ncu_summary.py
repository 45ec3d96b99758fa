"""Key metrics of every kernel in an ncu report (`--page details`)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(k) for k in
                          ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    cur = None
    for r in rows[1:]:
        if r[ii] != cur:
            cur = r[ii]
            print(f"== [{cur}] {r[ki][:90]}")
        if r[mi] in WANT:
            print(f"   {r[mi]:34s} {r[vi]} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1])
