#!/usr/bin/env bash
# round-2 GPU pass A: full GPU suite (incl. full-size goldens and the reference
# suite through the plugin), the bench line and the reference arm.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rf > gpurun_out/a_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/a_gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
echo "bench rc=$?" >> gpurun_out/a_bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/a_bench_ref.json 2> gpurun_out/a_bench_ref.err
echo "ref rc=$?" >> gpurun_out/a_bench_ref.err
