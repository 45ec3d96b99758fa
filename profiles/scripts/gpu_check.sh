#!/bin/bash
# One GPU round trip: tests, smoke, bench (+ A/B env), ncu launch list with
# DRAM bytes, one --set full capture of a named kernel. Outputs in gpurun_out/.
#   bash profiles/scripts/gpu_check.sh [tests|bench|ncu|full:<kernel regex>] ...
set -u
mkdir -p gpurun_out
for step in "$@"; do
  case "$step" in
    tests)
      timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
      echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
      echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json ;;
    bench:*)
      # bench:NAME=VAL -- the same with one environment switch
      kv="${step#bench:}"
      env "$kv" timeout 900 python bench.py --no-cpu-baseline > "gpurun_out/bench_${kv}.json" 2> "gpurun_out/bench_${kv}.err"
      echo "bench $kv rc=$?"; python -c "import json,sys; d=json.load(open(sys.argv[1])); print(d['value'], d['e2e']['value'] if d.get('e2e') else None, json.dumps(d['roofline']['stages']))" "gpurun_out/bench_${kv}.json" ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv \
        python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
      echo "ncu rc=$?"
      python profiles/traffic_summary.py gpurun_out/traffic.csv > gpurun_out/traffic.json && head -c 400 gpurun_out/traffic.json ;;
    fullk:*)
      rest="${step#fullk:}"; k="${rest%%:*}"; skip="${rest##*:}"
      timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip $skip -c 1 \
        -o "gpurun_out/full_${k//[^a-zA-Z0-9_]/_}_$skip" -f \
        python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/ncu_full.log" 2>&1
      echo "ncu full $k skip $skip rc=$?" ;;
    full:*)
      k="${step#full:}"
      timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 \
        -o "gpurun_out/full_${k//[^a-zA-Z0-9_]/_}" -f \
        python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/ncu_full.log" 2>&1
      echo "ncu full $k rc=$?" ;;
  esac
done
# (appended) fullk:<regex>:<skip> -- --set full of the (skip+1)-th matching launch
