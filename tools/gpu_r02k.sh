#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/panel_lab.py --scale 1.0 --W 12288 --R 8192 > gpurun_out/k_lab4.log 2>&1
echo "rc=$?" >> gpurun_out/k_lab4.log
timeout 900 python tools/panel_lab.py --scale 1.0 --W 14336 --R 4096 > gpurun_out/k_lab5.log 2>&1
echo "rc=$?" >> gpurun_out/k_lab5.log
