#!/usr/bin/env bash
# round-2 GPU pass FD: L2 policy of the gathered vectors' stores (xe evict_last, y evict_first), alternating processes
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/fd_l2pol.log
for r in 1 2; do
  for v in product l2pol_xe_last1 l2pol_y_ef1 l2pol_both; do
    if [ $v = product ]; then timeout 600 python tools/lib_ab.py >> gpurun_out/fd_l2pol.log 2>&1
    else PDHG_B200_LIB=tools/_libs/$v.so timeout 600 python tools/lib_ab.py >> gpurun_out/fd_l2pol.log 2>&1; fi
  done
done
echo "rc=$?" >> gpurun_out/fd_l2pol.log
