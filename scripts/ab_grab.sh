#!/bin/bash
TAG=${1:-abg}
for rep in 1 2; do
  for w in roadnet amazon0601 products; do
    for v in D E; do
      GCNB_LIB=paper_2212_05009_b200/lib/ab_$v.so timeout 900 python bench.py --workload $w --steps 20 --warmup 5 \
        --kernels-only > gpurun_out/${TAG}_${w}_${v}_r$rep.json 2> gpurun_out/${TAG}_${w}_${v}_r$rep.err
      echo "$w lib=$v rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_${v}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k if n.startswith(("fwd", "bwd"))})' 2>&1 | tail -1)"
    done
  done
done
