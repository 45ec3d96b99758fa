#!/bin/bash
# compute-sanitizer passes over the path (logs in gpurun_out/sanitize_*.log).
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, cases...
  local tool=$1; shift
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
    python profiles/sanitize_case.py "$@" > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|errors' gpurun_out/sanitize_${tool}.log | tail -2 | tr '\n' ' ')"
}
run memcheck nano config1 c2div4 m3div4
run racecheck nano config1
run synccheck nano config1
run initcheck nano config1
# the fused pyramid exchange: two processes mapping each other's pyramids
timeout 1500 $CS --tool memcheck --target-processes all --error-exitcode 9 \
  python -m pytest tests/test_gpu_exchange.py -q -x > gpurun_out/sanitize_exchange.log 2>&1
echo "exchange memcheck rc=$?: $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_exchange.log | tail -3 | tr '\n' ' ')"
