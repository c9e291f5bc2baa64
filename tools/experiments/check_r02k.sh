set -u
o=gpurun_out/c11; mkdir -p $o
timeout 600 python tools/tc_bench.py --only ru_b64_cfg2,ru_b64_half,ru_b128_mid,qrb_update > $o/tc_bench.jsonl 2> $o/tc_bench.err
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_drivers.py -m gpu -x -q > $o/gputest.log 2>&1; tail -2 $o/gputest.log
for c in cfg2 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err
done
