#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_2603_03150_b200/libpdhg_b200.so tools/_libs/libpdhg_bps6.so tools/_libs/libpdhg_bps8.so paper_2603_03150_b200/libpdhg_b200.so; do
  timeout 600 python tools/check_time.py --lib $lib >> gpurun_out/l_check.log 2>&1
done
echo "rc=$?" >> gpurun_out/l_check.log
