#!/usr/bin/env bash
# round-2 GPU pass FM: check fusion under a numerical failure
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_check_fuse.py -m gpu -q -p no:cacheprovider --timeout 600 -rfs > gpurun_out/fm_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fm_tests.log
