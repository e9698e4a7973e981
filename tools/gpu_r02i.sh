#!/usr/bin/env bash
# round-2 GPU pass I: bounds-checked workload, full GPU suite, experiment-build parity, bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PDHG_B200_LIB=$PWD/tools/_libs/libpdhg_b200_checked.so timeout 1200 python tools/sanitize_run.py > gpurun_out/i_bounds.log 2>&1
echo "bounds rc=$?" >> gpurun_out/i_bounds.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs > gpurun_out/i_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/i_gpu_tests.log
PDHG_B200_LIB=$PWD/tools/_libs/libpdhg_b200_exp.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "psr or persistent or tiny" > gpurun_out/i_exp_tests.log 2>&1
echo "exp tests rc=$?" >> gpurun_out/i_exp_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
echo "bench rc=$?" >> gpurun_out/i_bench.err
