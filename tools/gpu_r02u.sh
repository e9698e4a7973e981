#!/usr/bin/env bash
# round-2 GPU pass U (re-entry): HEAD suite, smoke, bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs --durations=25 > gpurun_out/u_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/u_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/u_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/u_bench.json 2> gpurun_out/u_bench.err
echo "bench rc=$?" >> gpurun_out/u_bench.err
