#!/usr/bin/env bash
# round-2 GPU pass Y: the multi-GPU bench path on a world of one (--sharded), NCCL and peer
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --sharded --scale 0.05 --steps 3 --warmup 3 --no-cpu > gpurun_out/y_sharded_nccl.json 2> gpurun_out/y_sharded_nccl.err
echo "rc=$?" >> gpurun_out/y_sharded_nccl.err
timeout 900 python bench.py --sharded --comm peer --scale 0.05 --steps 3 --warmup 3 --no-cpu > gpurun_out/y_sharded_peer.json 2> gpurun_out/y_sharded_peer.err
echo "rc=$?" >> gpurun_out/y_sharded_peer.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --sharded --scale 1.0 --steps 3 --warmup 3 --no-cpu > gpurun_out/y_sharded_full.json 2> gpurun_out/y_sharded_full.err
echo "rc=$?" >> gpurun_out/y_sharded_full.err
