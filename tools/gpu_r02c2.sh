#!/usr/bin/env bash
# round-2 GPU pass C2: x-space (column) renumbering -- A/B, full GPU suite, bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python tools/ab_layout.py --variants rows,rows_nocol --rounds 10 > gpurun_out/c_ab.log 2>&1
echo "ab rc=$?" >> gpurun_out/c_ab.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs --durations=10 > gpurun_out/c_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/c_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
echo "bench rc=$?" >> gpurun_out/c_bench.err
