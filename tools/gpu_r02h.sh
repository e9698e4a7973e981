#!/usr/bin/env bash
# round-2 GPU pass H: compute-sanitizer memcheck / racecheck / synccheck over the workload
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/sanitize_run.py > gpurun_out/h_plain.log 2>&1
echo "plain rc=$?" >> gpurun_out/h_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > gpurun_out/h_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/h_$tool.log
done
