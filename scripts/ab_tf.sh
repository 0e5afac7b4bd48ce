#!/bin/bash
TAG=${1:-tf}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_path.py tests/test_gpu_configs.py tests/test_gpu_races.py -q -x > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/${TAG}_tests.log)"
for rep in 1 2; do
  for w in ${WLS:-roadnet amazon0601 config1}; do
    for v in 0 1; do
      GCNB_FWD_TF=$v timeout 900 python bench.py --workload $w --steps 20 --warmup 5 \
        --kernels-only > gpurun_out/${TAG}_${w}_${v}_r$rep.json 2> gpurun_out/${TAG}_${w}_${v}_r$rep.err
      echo "$w tf=$v rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_${v}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_step"], {n: k[n]["ms_per_launch"] for n in k if n.startswith(("fwd", "bwd"))})' 2>&1 | tail -1)"
    done
  done
done
