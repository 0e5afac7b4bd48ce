#!/bin/bash
# 1-GPU bench lines of every workload (device + the reference arm on the host cores).
# usage (under gpurun): bash scripts/n1_sweep.sh tag
TAG=${1:-n1}
mkdir -p gpurun_out
for w in config1 amazon0601 roadnet; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/${TAG}_${w}_n1.json 2> gpurun_out/${TAG}_${w}_n1.err
  echo "$w rc=$? $(tail -1 gpurun_out/${TAG}_${w}_n1.json | cut -c1-120)"
  timeout 900 python bench.py --impl reference --workload $w --steps 5 --warmup 1 > gpurun_out/${TAG}_${w}_ref.json 2> gpurun_out/${TAG}_${w}_ref.err
  echo "$w reference rc=$? $(tail -1 gpurun_out/${TAG}_${w}_ref.json | cut -c1-120)"
done
