#!/usr/bin/env bash
# round-2 GPU pass FC: quad gather load shapes of the fused dual step (256-bit, 2x128-bit, 256-bit no-L1-allocate)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 1 2; do
  PDHG_B200_LIB=tools/_libs/quad_ld$v.so timeout 600 python tools/check_fuse_ab.py --rounds 6 > gpurun_out/fc_ab_ld$v.log 2>&1
  echo "ab rc=$?" >> gpurun_out/fc_ab_ld$v.log
done
timeout 600 python tools/check_fuse_ab.py --rounds 6 > gpurun_out/fc_ab_ld0.log 2>&1
echo "ab rc=$?" >> gpurun_out/fc_ab_ld0.log
for v in 1 2; do
  PDHG_B200_LIB=tools/_libs/quad_ld$v.so timeout 600 ncu --clock-control none -k regex:k_step_sell_chk -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --csv python bench.py --steps 1 --warmup 3 --no-cpu --no-ttk > gpurun_out/fc_ncu_ld$v.csv 2>&1
done
