#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pass in 1 2; do
for lib in paper_2603_03150_b200/libpdhg_b200.so tools/_libs/libpdhg_PDHG_SELL_U_LONG_8.so tools/_libs/libpdhg_PDHG_SELL_U_LONG_8_PDHG_SELL_MINB_6.so tools/_libs/libpdhg_PDHG_SELL_U_LONG_10_PDHG_SELL_MINB_6.so tools/_libs/libpdhg_PDHG_SELL_U_LONG_4.so; do
  PDHG_B200_LIB=$PWD/$lib timeout 600 python tools/lib_ab.py --scale 0.5 >> gpurun_out/p_libs.log 2>&1
done
done
echo "rc=$?" >> gpurun_out/p_libs.log
