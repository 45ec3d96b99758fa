#!/bin/bash
# A/B of one kernel family's serialised time between library builds, with a
# substring filter on the demangled name (template arguments included):
#   ab_family.sh <ncu -k regex> <name substring> <lib1> <lib2> ...
k=$1; sub=$2; shift 2
for lib in "$@"; do
  rm -f /tmp/ab.csv
  LVSG_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$k" --csv \
    --log-file /tmp/ab.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.log 2>&1 \
    || { echo "$lib: run failed"; tail -3 /tmp/ab.log; continue; }
  python - "$lib" "$sub" <<'PY'
import csv, sys
lines=[l for l in open('/tmp/ab.csv') if l.startswith('"')]
rows=list(csv.reader(lines)); h=rows[0]; vi=h.index('Metric Value'); ki=h.index('Kernel Name')
v=[float(r[vi].replace(',',''))/1e3 for r in rows[1:] if sys.argv[2] in r[ki]]
print(sys.argv[1], 'launches', len(v), 'us per frame', round(sum(v) / 7, 1), 'last', [round(x, 1) for x in v[-10:]])
PY
done
