#!/usr/bin/env bash
# round-2 GPU pass FA: check fused into the last dual step -- parity tests, interleaved A/B (unroll variants), bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_check_fuse.py tests/test_gpu_check_dot.py tests/test_native_abi.py -q -p no:cacheprovider --timeout 900 -rfs -x > gpurun_out/fa_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fa_tests.log
timeout 600 python tools/check_fuse_ab.py --rounds 8 > gpurun_out/fa_ab_u4.log 2>&1
echo "ab rc=$?" >> gpurun_out/fa_ab_u4.log
for u in 6 8; do
  PDHG_B200_LIB=tools/_libs/fuse_u$u.so timeout 600 python tools/check_fuse_ab.py --rounds 6 > gpurun_out/fa_ab_u$u.log 2>&1
  echo "ab rc=$?" >> gpurun_out/fa_ab_u$u.log
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fa_bench.json 2> gpurun_out/fa_bench.err
echo "bench rc=$?" >> gpurun_out/fa_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/fa_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-ttk > gpurun_out/fa_ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/fa_ncu_list.log
