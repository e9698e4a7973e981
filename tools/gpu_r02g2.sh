#!/usr/bin/env bash
# round-2 GPU pass G2: pooled streams -- setup profile, full GPU suite, bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/setup_profile.py > gpurun_out/g_setup.log 2>&1
echo "rc=$?" >> gpurun_out/g_setup.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs --durations=10 > gpurun_out/g_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
echo "bench rc=$?" >> gpurun_out/g_bench.err
