set -u
o=gpurun_out/c10; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/gputest.log 2>&1; tail -2 $o/gputest.log
timeout 600 python tools/tc_bench.py > $o/tc_bench.jsonl 2> $o/tc_bench.err
for c in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err
done
