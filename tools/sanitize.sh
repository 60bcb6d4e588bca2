#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
# (PDL on).  Logs -> gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --target-processes all \
    python tools/sanitize_run.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
