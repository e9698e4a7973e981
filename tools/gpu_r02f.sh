#!/usr/bin/env bash
# round-2 GPU pass F: interleaved layout A/B + overlap tests
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python tools/ab_layout.py --variants natural,rows,rows_csr,csr --rounds 8 > gpurun_out/f_ab.log 2>&1
echo "ab rc=$?" >> gpurun_out/f_ab.log
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider -x -k "overlap" > gpurun_out/f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/f_tests.log
