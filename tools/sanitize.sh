#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (small c1, c2, c4,
# c6 DAGs through the dataflow, op-by-op and Ozaki executors, values checked against the oracle).
# Output: gpurun_out/sanitize_<tool>.log (summaries copied to profiles/ by hand).
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout -s KILL ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --print-limit 50 \
    python tools/sanitize_run.py ${SAN_ARGS} > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
