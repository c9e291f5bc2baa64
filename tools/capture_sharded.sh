#!/bin/bash
# world-1 NCCL runs of the sharded drivers (one GPU per gpurun)
o=gpurun_out/x; mkdir -p $o
for c in cfg2 cfg3 cfg5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --force-sharded --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $o/sharded_$c.json 2> $o/sharded_$c.err
  tail -c 300 $o/sharded_$c.json; echo
done
