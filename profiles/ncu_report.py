"""Text summary of an ncu --set full report for profiles/: per kernel the
duration, DRAM bytes per launch (the roofline `traffic`), throughput
fractions, pipe utilisation, occupancy and the top stall lines."""
import csv
import io
import subprocess
import sys

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main(rep, title=""):
    print(f"# {title or rep}")
    for vals, units in raw(rep):
        print(f"\n## {vals.get('Kernel Name', '?')[:110]}")
        for key, label in RAW:
            if key in vals:
                print(f"  {label:24s} {vals[key]} {units.get(key, '')}")
    print()
    sys.stdout.flush()
    subprocess.run([sys.executable, __file__.replace("ncu_report.py", "source_hotspots.py"), rep, "12"])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
