set -u
o=gpurun_out/c7; mkdir -p $o
for c in cfg5 cfg2 cfg3; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --config $c --force-sharded --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $o/sharded_$c.json 2> $o/sharded_$c.err
done
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -x -q > $o/gputest_sharded.log 2>&1; tail -2 $o/gputest_sharded.log
