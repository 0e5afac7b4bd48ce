#!/bin/bash
# ncu evidence for the default bench workload (1 GPU): plain run, launch list, full capture of one epoch.
# usage (under gpurun): bash scripts/profile_products.sh [workload] [tag]
set -e
WL=${1:-products}; TAG=${2:-r01}
CMD="python bench.py --workload $WL --steps 1 --warmup 3 --kernels-only"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_${WL}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/${TAG}_${WL}_launches.csv $CMD > gpurun_out/${TAG}_${WL}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -s 16 -c 16 \
    -o gpurun_out/${TAG}_${WL}_full $CMD > gpurun_out/${TAG}_${WL}_ncu_full.log 2>&1
