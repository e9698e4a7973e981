#!/usr/bin/env bash
# round-2 GPU pass F: long-rows-first renumbering -- full GPU suite, bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs --durations=15 > gpurun_out/f_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/f_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
echo "bench rc=$?" >> gpurun_out/f_bench.err
