#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider -k "torch_peer or torch_comm or fused" > gpurun_out/m_tests.log 2>&1
echo "rc=$?" >> gpurun_out/m_tests.log
