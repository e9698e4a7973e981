set -x
python -m pytest tests -m gpu -x -q > gpurun_out/v14_tests.log 2>&1; tail -1 gpurun_out/v14_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v14_smoke.log 2>&1; tail -1 gpurun_out/v14_smoke.log
python bench.py > gpurun_out/v14_bench.json 2> gpurun_out/v14_bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/v14_ref.json 2> gpurun_out/v14_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/v14_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/v14_ncu.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_step|k_check" -s 300 -c 4 -o gpurun_out/v14_full python bench.py --steps 2 --warmup 1 --no-cpu --no-ttk > gpurun_out/v14_full.log 2>&1; echo ncu2 rc=$?
