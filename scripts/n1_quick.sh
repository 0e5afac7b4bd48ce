#!/bin/bash
# 1-GPU kernel tests + bench lines for the small workloads and products (no reference arm).
# usage (under gpurun): bash scripts/n1_quick.sh tag [tests]
TAG=${1:-nq}
mkdir -p gpurun_out
if [ "${2:-tests}" = "tests" ]; then
  timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_races.py tests/test_gpu_path.py -q -x \
    > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/${TAG}_tests.log)"
fi
for w in amazon0601 roadnet config1 products; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-products3 > gpurun_out/${TAG}_${w}_n1.json 2> gpurun_out/${TAG}_${w}_n1.err
  echo "$w rc=$? $(tail -1 gpurun_out/${TAG}_${w}_n1.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k: v["ms_per_launch"] for k, v in d["kernels"].items()})' 2>&1 | tail -1)"
done
