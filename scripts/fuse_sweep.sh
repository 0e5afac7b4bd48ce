#!/bin/bash
# Fused halo packs (producer epilogues) vs separate pack kernels, one process per GPU.
# usage (under gpurun --gpus N): bash scripts/fuse_sweep.sh tag [tests]
TAG=${1:-fz}
mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
if [ "${2:-tests}" = "tests" ]; then
  timeout 1200 python -m pytest tests/test_gpu_distributed.py -q > gpurun_out/${TAG}_dist_tests.log 2>&1
  echo "dist tests rc=$? $(tail -1 gpurun_out/${TAG}_dist_tests.log)"
  timeout 600 python -m pytest tests/test_gpu_path.py -q -k "threads or deterministic" > gpurun_out/${TAG}_threads.log 2>&1
  echo "threads tests rc=$? $(tail -1 gpurun_out/${TAG}_threads.log)"
fi
run() {  # workload partition fuse
  local w=$1 p=$2 f=$3
  GCNB_FUSE_PACK=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --workload $w --partition $p \
    > gpurun_out/${TAG}_${w}_n${n}_${p}_f${f}_r${rep}.json 2> gpurun_out/${TAG}_${w}_n${n}_${p}_f${f}_r${rep}.err
  echo "$w n=$n $p fuse=$f rep=$rep rc=$? $(tail -1 gpurun_out/${TAG}_${w}_n${n}_${p}_f${f}_r${rep}.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d.get("exposed_comm_pct"), d.get("e2e", {}).get("value"))' 2>&1 | tail -1)"
}
for rep in 1 2; do
  for w in amazon0601 roadnet products; do
    for f in 0 1 2; do run $w hp-ml $f; done
  done
done
