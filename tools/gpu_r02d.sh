#!/usr/bin/env bash
# round-2 GPU pass D: ncu of the step + check kernels (renumbered-rows SELL), launch list
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -k "rows" > gpurun_out/d_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/d_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/d_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/d_ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/d_ncu_list.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_step|k_check' -s 300 -c 5 -o gpurun_out/d_full -f python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/d_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/d_ncu_full.log
