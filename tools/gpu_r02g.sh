#!/usr/bin/env bash
# round-2 GPU pass G: epilogue cache policy A/B (+ DRAM bytes under ncu)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python tools/ab_layout.py --variants rows,rows_cs,natural,natural_cs --rounds 8 > gpurun_out/g_ab.log 2>&1
echo "ab rc=$?" >> gpurun_out/g_ab.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_step -c 8 --csv python tools/ab_layout.py --variants rows,rows_cs --rounds 1 > gpurun_out/g_ncu.csv 2> gpurun_out/g_ncu.err
echo "ncu rc=$?" >> gpurun_out/g_ncu.err
