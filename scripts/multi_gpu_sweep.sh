#!/bin/bash
# Multi-GPU measurements (one process per GPU, torchrun): products at 2/4 GPUs,
# roadNet HP vs GP vs RP (BASELINE config[2]) and amazon0601 at 4 GPUs.
# usage (under gpurun --gpus 4): bash scripts/multi_gpu_sweep.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
run() {  # n workload partition
  local n=$1 w=$2 p=$3
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --workload $w --partition $p \
    > gpurun_out/${TAG}_${w}_n${n}_${p}.json 2> gpurun_out/${TAG}_${w}_n${n}_${p}.err
  echo "$w n=$n $p rc=$? $(tail -1 gpurun_out/${TAG}_${w}_n${n}_${p}.json | cut -c1-160)"
}
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/${TAG}_dist_tests.log 2>&1
echo "dist tests rc=$? $(tail -1 gpurun_out/${TAG}_dist_tests.log)"
run 4 products hp-ml
run 2 products hp-ml
run 4 roadnet hp-ml
run 4 roadnet gp-ml
run 4 roadnet rp
run 4 amazon0601 hp-ml
