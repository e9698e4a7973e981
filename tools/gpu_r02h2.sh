#!/usr/bin/env bash
# round-2 GPU pass H2: epilogue cache policy A/B (product lib vs PDHG_EPI_HINT=1), one process per lib, alternating
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/h_epi.log
for r in 1 2 3; do
  timeout 300 python tools/lib_ab.py >> gpurun_out/h_epi.log 2>&1
  PDHG_B200_LIB=tools/_libs/libpdhg_b200_epi.so timeout 300 python tools/lib_ab.py >> gpurun_out/h_epi.log 2>&1
done
echo done >> gpurun_out/h_epi.log
