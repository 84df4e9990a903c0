# Two ranks on ONE GPU with the gloo backend: exercises bench.py's N>1 code
# paths (batch-shard cfg2, vocab-shard cfg4 with the record all-gather,
# batch-shard cfg3) the driver's NCCL scaling run uses; not a scaling number.
export SVT_DIST_BACKEND=gloo
for w in ${WORKLOADS:-cfg2 cfg4 cfg3}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 1 --workload $w --no-secondary \
    --no-cpu-baseline --no-e2e > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "$w rc=$?" >> gpurun_out/mr.log
done
