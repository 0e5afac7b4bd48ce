#!/bin/bash
# A/B of library builds (GCNB_LIB) on one box, interleaved: bench --kernels-only per workload.
# usage (under gpurun): bash scripts/ab_libs.sh tag "A B C" "roadnet amazon0601 products" [reps]
TAG=$1; VARS=$2; WLS=$3; REPS=${4:-2}
mkdir -p gpurun_out
for rep in $(seq 1 $REPS); do
  for w in $WLS; do
    for v in $VARS; do
      GCNB_LIB=paper_2212_05009_b200/lib/ab_$v.so timeout 900 python bench.py --workload $w --steps 20 --warmup 5 \
        --kernels-only > gpurun_out/${TAG}_${w}_${v}_r$rep.json 2> gpurun_out/${TAG}_${w}_${v}_r$rep.err
      echo "$w $v rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_${v}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k if n.startswith(("fwd", "bwd"))})' 2>&1 | tail -1)"
    done
  done
done
