timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/r2s13_dist.log 2>&1; echo "dist rc=$? $(tail -1 gpurun_out/r2s13_dist.log)"
for w in amazon0601 roadnet; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --workload $w --partition hp-ml > gpurun_out/r2s13_${w}_n4.json 2> gpurun_out/r2s13_${w}_n4.err
  echo "$w rc=$?"
done
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29777 scripts/dist_minibatch.py --vertices 4194304 --batch 1048576 --steps 6 > gpurun_out/r2s13_dmb.json 2> gpurun_out/r2s13_dmb.err; echo "dmb rc=$?"
