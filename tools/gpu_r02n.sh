#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/config2_full.py > gpurun_out/n_config2.log 2>&1
echo "rc=$?" >> gpurun_out/n_config2.log
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider > gpurun_out/n_configs.log 2>&1
echo "rc=$?" >> gpurun_out/n_configs.log
