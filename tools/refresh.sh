#!/bin/bash
# Round-end refresh: GPU tests, bench lines for every config, reference arm,
# and the ncu launch list of the cfg2 bench command.  Outputs in gpurun_out/g.
set -u
o=gpurun_out/g; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c > $o/bench_$c.json 2> $o/bench_$c.err
done
timeout 300 python bench.py --impl reference > $o/bench_ref_cfg2.json 2> $o/bench_ref_cfg2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include timed/ \
  --csv --log-file $o/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e > $o/ncu_launch.log 2>&1
tail -c 300 $o/bench_*.json
