#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
echo "bench rc=$?" >> gpurun_out/s_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_check' -c 4 -o gpurun_out/s_check -f python bench.py --steps 1 --warmup 1 --no-cpu --no-ttk > gpurun_out/s_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s_ncu.log
