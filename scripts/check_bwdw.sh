#!/bin/bash
TAG=${1:-bw}
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_path.py tests/test_gpu_configs.py tests/test_gpu_races.py -q -x > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/${TAG}_tests.log)"
for rep in 1 2; do
  for w in config1 amazon0601 roadnet; do
    for v in 0 1; do
      GCNB_BWD_WARP=$v timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --kernels-only > gpurun_out/${TAG}_${w}_${v}_r$rep.json 2> gpurun_out/${TAG}_${w}_${v}_r$rep.err
      echo "$w bwdw=$v rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_${v}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k if n.startswith(("fwd", "bwd", "reduce"))})' 2>&1 | tail -1)"
    done
  done
done
CMD="python bench.py --steps 3 --warmup 3 --kernels-only --no-products3"
$CMD > gpurun_out/${TAG}_plain.json 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$? $(grep -c '^\"' gpurun_out/${TAG}_launches.csv)"
