#!/bin/bash
# interleaved A/B of two library builds (lib/ab_A.so, lib/ab_B.so) on the given workloads
TAG=${1:-ab}; WLS=${2:-"config1 amazon0601 roadnet"}
for rep in 1 2; do
  for w in $WLS; do
    for v in A B; do
      GCNB_LIB=paper_2212_05009_b200/lib/ab_$v.so timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --kernels-only > gpurun_out/${TAG}_${w}_${v}_r$rep.json 2> gpurun_out/${TAG}_${w}_${v}_r$rep.err
      echo "$w $v rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_${v}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k if n.startswith(("fwd", "bwd"))})' 2>&1 | tail -1)"
    done
  done
done
