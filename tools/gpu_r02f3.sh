#!/usr/bin/env bash
# round-2 GPU pass F2: final-state (16k windows) launch list + ncu --set full of the step and check kernels
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/f2_ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/f2_ncu_list.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_step|k_check|k_primal_from' -s 300 -c 10 -o gpurun_out/f2_full -f python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/f2_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/f2_ncu_full.log
