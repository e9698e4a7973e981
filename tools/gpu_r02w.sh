#!/usr/bin/env bash
# round-2 GPU pass W: product step kernels vs minimal SELL SpMV on the same layouts
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/sell_lab.py --rounds 5 > gpurun_out/w_sell_lab.log 2>&1
echo "rc=$?" >> gpurun_out/w_sell_lab.log
