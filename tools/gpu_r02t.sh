#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/t_hostio.log; timeout 300 python tools/hostio_lab.py >> gpurun_out/t_hostio.log 2>&1
echo "rc=$?" >> gpurun_out/t_hostio.log
