#!/bin/bash
# bench --kernels-only lines for the given workloads (2 reps), env passed through.
TAG=${1:-q}; WLS=${2:-"config1 amazon0601 roadnet"}
for rep in 1 2; do
  for w in $WLS; do
    timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --kernels-only > gpurun_out/${TAG}_${w}_r$rep.json 2> gpurun_out/${TAG}_${w}_r$rep.err
    echo "$w rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k if n.startswith(("fwd", "bwd"))})' 2>&1 | tail -1)"
  done
done
