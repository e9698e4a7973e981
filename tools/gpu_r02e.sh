#!/usr/bin/env bash
# round-2 GPU pass E: full GPU suite on the product build + bench + smoke
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs > gpurun_out/e_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/e_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/e_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
echo "bench rc=$?" >> gpurun_out/e_bench.err
