#!/usr/bin/env bash
# round-2 GPU pass FZ: final state -- full suite, smoke, bench, reference arm, launch list, ncu of the step / check kernels
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfs --durations=10 > gpurun_out/fz_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fz_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fz_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fz_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fz_bench.json 2> gpurun_out/fz_bench.err
echo "bench rc=$?" >> gpurun_out/fz_bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/fz_bench_ref.json 2> gpurun_out/fz_bench_ref.err
echo "ref rc=$?" >> gpurun_out/fz_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/fz_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-ttk > gpurun_out/fz_ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/fz_ncu_list.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_step|k_check|k_primal_from' -s 300 -c 12 -o gpurun_out/fz_full -f python bench.py --steps 2 --warmup 3 --no-cpu --no-ttk > gpurun_out/fz_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/fz_ncu_full.log
