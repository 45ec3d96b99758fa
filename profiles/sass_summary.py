"""Per-kernel SASS evidence of the Blackwell paths: counts of the tcgen05 /
TMA / TMEM mnemonics (B200_PROFILING.md: UTCHMMA = tcgen05.mma, UTMALDG /
UTMASTG = TMA tensor load / store, UBLKCP = cp.async.bulk, LDTM / STTM =
tcgen05.ld / st, UTCBAR = tcgen05.commit) in every kernel of liblvsg.so.

  python profiles/sass_summary.py > profiles/r2/sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2411_16680_b200", "liblvsg.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR",
        "SYNCS", "DFMA", "DMUL", "LDG", "STG", "LDS", "STS"]


def demangle(names):
    p = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return p.stdout.splitlines() if p.returncode == 0 else names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else LIB
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    kern = None
    counts = collections.OrderedDict()
    total = collections.Counter()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and kern:
            op = m.group(2)
            counts[kern]["_insts"] += 1
            for k in KEYS:
                if op == k or op.startswith(k):
                    counts[kern][k] += 1
                    break
    names = demangle(list(counts))
    print(f"# SASS mnemonic counts per kernel in {os.path.relpath(lib, ROOT)} (sm_100a)")
    print("# static instruction counts; UTCHMMA = tcgen05.mma, UTMALDG/UTMASTG = TMA, "
          "LDTM = tcgen05.ld, UBLKCP = cp.async.bulk")
    hdr = ["insts"] + KEYS
    print(f"{'kernel':<90} " + " ".join(f"{h:>7}" for h in hdr))
    for (k, c), n in zip(counts.items(), names):
        short = re.sub(r"lvsg::\(anonymous namespace\)::|lvsg::", "", n)
        short = short if len(short) <= 90 else short[:87] + "..."
        print(f"{short:<90} " + " ".join(f"{c.get('_insts' if h == 'insts' else h, 0):>7}"
                                         for h in hdr))
        total.update(c)
    print(f"{'TOTAL':<90} " + " ".join(f"{total.get('_insts' if h == 'insts' else h, 0):>7}"
                                       for h in hdr))


if __name__ == "__main__":
    main()
