#!/bin/bash
# A/B: library variants and GCNB_SPLIT_ALL on the small workloads and products (1 GPU).
TAG=${1:-abs}
for rep in 1 2; do
  for w in roadnet amazon0601; do
    for cfg in "C 0" "C 1" "D 0"; do
      set -- $cfg
      GCNB_LIB=paper_2212_05009_b200/lib/ab_$1.so GCNB_SPLIT_ALL=$2 timeout 900 python bench.py --workload $w --steps 20 --warmup 5 \
        --kernels-only > gpurun_out/${TAG}_${w}_$1_s$2_r$rep.json 2> gpurun_out/${TAG}_${w}_$1_s$2_r$rep.err
      echo "$w lib=$1 split=$2 rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_$1_s$2_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k})' 2>&1 | tail -1)"
    done
  done
  for v in C D; do
    GCNB_LIB=paper_2212_05009_b200/lib/ab_$v.so timeout 900 python bench.py --workload products --steps 20 --warmup 5 \
      --kernels-only > gpurun_out/${TAG}_products_${v}_r$rep.json 2> gpurun_out/${TAG}_products_${v}_r$rep.err
    echo "products lib=$v rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_products_${v}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k if n.startswith(("fwd", "bwd2"))})' 2>&1 | tail -1)"
  done
done
