#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pass in 1 2 3; do
for lib in paper_2603_03150_b200/libpdhg_b200.so tools/_libs/libpdhg_dual_u6.so; do
  PDHG_B200_LIB=$PWD/$lib timeout 600 python tools/lib_ab.py --scale 1.0 >> gpurun_out/q_libs.log 2>&1
done
done
echo "rc=$?" >> gpurun_out/q_libs.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_bounds.py -m gpu -q -p no:cacheprovider -x > gpurun_out/q_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/q_tests.log
