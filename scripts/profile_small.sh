#!/bin/bash
# ncu of the narrow-layer kernels on a small graph (1 GPU): plain run, then a full capture of the first epoch.
# usage (under gpurun): bash scripts/profile_small.sh [workload] [tag]
WL=${1:-roadnet}; TAG=${2:-ps}
CMD="python bench.py --workload $WL --steps 1 --warmup 3 --kernels-only"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_${WL}_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_gemm|k_bwd|k_agg|k_loss|k_dense" -c 8 \
    -o gpurun_out/${TAG}_${WL}_full $CMD > gpurun_out/${TAG}_${WL}_ncu_full.log 2>&1; echo "ncu rc=$?"
