#!/bin/bash
# compute-sanitizer over tools/sanitize.py; logs to gpurun_out/sanitize_<tool>.log
set -u
mkdir -p gpurun_out
timeout 600 python tools/sanitize.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/sanitize_plain.log
for tool in memcheck synccheck racecheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize.py --quick > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
