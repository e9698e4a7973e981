#!/usr/bin/env bash
# round-2 GPU pass V: gather4 / 128-bit stream lab (tools/gather4_lab.cu)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/v_lab.log 2>&1
timeout 300 tools/gather4_lab 5000000 40 20 >> gpurun_out/v_lab.log 2>&1
echo "rc=$?" >> gpurun_out/v_lab.log
timeout 300 tools/gather4_lab 5000000 40 20 >> gpurun_out/v_lab.log 2>&1
echo "rc=$?" >> gpurun_out/v_lab.log
