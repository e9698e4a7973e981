#!/usr/bin/env bash
# round-2 GPU pass FB: full GPU suite with the fused check, occupancy variants of the fused dual step, ncu of it
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs --durations=10 > gpurun_out/fb_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fb_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fb_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fb_smoke.log
for v in u3_b6 u4_b6; do
  PDHG_B200_LIB=tools/_libs/fuse_$v.so timeout 600 python tools/check_fuse_ab.py --rounds 6 > gpurun_out/fb_ab_$v.log 2>&1
  echo "ab rc=$?" >> gpurun_out/fb_ab_$v.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_step_sell_chk|k_check_primal_fold|k_check_dual_sell' -c 3 -o gpurun_out/fb_full -f python bench.py --steps 2 --warmup 3 --no-cpu --no-ttk > gpurun_out/fb_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/fb_ncu_full.log
