#!/usr/bin/env bash
# round-2 GPU pass FL: full GPU suite + smoke on the final code
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs --durations=10 > gpurun_out/fl_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fl_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fl_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fl_smoke.log
