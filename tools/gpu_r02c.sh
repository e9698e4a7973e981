#!/usr/bin/env bash
# round-2 GPU pass C: renumbered-rows SELL parity + kernel matrix + short bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "rows or full_size_against" -x > gpurun_out/c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/c_tests.log
timeout 1200 python tools/kernel_matrix.py --variants natural,rows,rows_w4k,rows_global,rows_h1k > gpurun_out/c_km.log 2>&1
echo "km rc=$?" >> gpurun_out/c_km.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
echo "bench rc=$?" >> gpurun_out/c_bench.err
