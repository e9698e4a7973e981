#!/usr/bin/env bash
# round-2 GPU pass B: window-sorted SELL parity + kernel matrix on config 4
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -k "window" -x > gpurun_out/b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/b_tests.log
timeout 1200 python tools/kernel_matrix.py --variants nowindow,window,window_h128,window_h192,window_h512 > gpurun_out/b_km.log 2>&1
echo "km rc=$?" >> gpurun_out/b_km.log
