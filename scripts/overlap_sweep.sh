#!/bin/bash
# Small graphs at N GPUs with and without the interior/boundary overlap.
# usage (under gpurun --gpus N): bash scripts/overlap_sweep.sh tag
TAG=${1:-ov}
n=$(nvidia-smi -L | wc -l)
for w in amazon0601 roadnet; do
  for ov in on off; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --workload $w --partition hp-ml --overlap $ov \
      > gpurun_out/${TAG}_${w}_n${n}_ov${ov}.json 2> gpurun_out/${TAG}_${w}_n${n}_ov${ov}.err
    python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_${w}_n${n}_ov${ov}.json').read().strip().splitlines()[-1])
print('$w', 'overlap=$ov', d['value'], 'exposed', d['exposed_comm_pct'], 'compute_only', d['compute_only_ms'])"
  done
done
