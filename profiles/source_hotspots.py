"""Per-CUDA-source-line warp-stall samples from an ncu report
(`ncu -i R --page source --csv --print-source sass,cuda`)."""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass,cuda"], capture_output=True, text=True).stdout
    fname, rows, total = None, [], 0
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif len(r) > 6 and r[0].isdigit():
            n = int(r[4]) if r[4].isdigit() else 0
            total += n
            rows.append((n, fname, int(r[0]), r[1].strip()))
    rows.sort(reverse=True)
    print(f"total samples {total}")
    for n, f, ln, src in rows[:top]:
        print(f"{n:7d} {100 * n / max(total, 1):5.1f}%  {f}:{ln}  {src[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
