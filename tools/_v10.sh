set -x
python -m pytest tests -m gpu -x -q > gpurun_out/v10_tests.log 2>&1; tail -3 gpurun_out/v10_tests.log
python bench.py > gpurun_out/v10_bench.json 2> gpurun_out/v10_bench.err; echo bench rc=$?
tail -c 600 gpurun_out/v10_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/v10_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/v10_ncu.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_step -s 300 -c 2 -o gpurun_out/v10_full python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/v10_full.log 2>&1; echo ncu2 rc=$?
