#!/bin/bash
# 2-GPU check: the torchrun parity tests, then the products bench at 2 GPUs.
# usage (under gpurun --gpus 2): bash scripts/dist_quick.sh tag
TAG=${1:-dq}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/${TAG}_dist_tests.log 2>&1
echo "dist tests rc=$? $(tail -1 gpurun_out/${TAG}_dist_tests.log)"
n=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
  --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --workload ${2:-products} --partition hp-ml \
  > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$? $(tail -1 gpurun_out/${TAG}_bench.json | cut -c1-200)"
