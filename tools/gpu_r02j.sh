#!/usr/bin/env bash
# round-2 GPU pass J: sharded tests (replay, overlap) + scaled/parity quick check
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider > gpurun_out/j_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/j_tests.log
