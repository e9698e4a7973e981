#!/usr/bin/env bash
# round-2 GPU pass FK: where a sharded period goes (loopback G=1, config 4), whole-row sliced ELL for the shards' check; sharded tests; world-1 bench
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/sharded_breakdown.py > gpurun_out/fk_breakdown.log 2>&1
echo "rc=$?" >> gpurun_out/fk_breakdown.log
timeout 1800 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider --timeout 1200 -rfs > gpurun_out/fk_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fk_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --sharded --scale 1.0 --steps 10 --warmup 3 --no-cpu > gpurun_out/fk_sharded_full.json 2> gpurun_out/fk_sharded_full.err
echo "rc=$?" >> gpurun_out/fk_sharded_full.err
