#!/bin/bash
# Round-2 measurement pass (one gpurun call): bench lines, reference arm,
# the ncu launch list of the cfg2 timed pass, DRAM traffic of the roofline
# kernel and one --set full capture of it.  Outputs in gpurun_out/r2.
set -u
o=${OUT:-gpurun_out/r2}; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/gputest.log 2>&1; tail -2 $o/gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $o/bench_ref_cfg2.json 2> $o/bench_ref_cfg2.err
for c in ${CONFIGS:-cfg3 cfg4 cfg5 cfg1}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $o/bench_$c.json 2> $o/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include timed/ \
  --csv --log-file $o/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e > $o/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:rank_update_grouped -c 200 --csv --log-file $o/traffic_update_cfg2.csv \
  python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $o/ncu_traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rank_update_grouped -s 20 -c 1 \
  -o $o/ncu_update_cfg2 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline \
  --no-e2e > $o/ncu_full.log 2>&1
tail -c 400 $o/bench_*.json
# the two latency-chain kernels (block ~60 of cfg2), one --set full capture each
for k in panel_fast_kernel select_reg_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 60 -c 1 \
    -o $o/ncu_${k}_cfg2 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline \
    --no-e2e > $o/ncu_full_$k.log 2>&1
done
# the dominant product of cfg3 (TRQRCP's G = Y_b^T A, tc_tma_kernel) and cfg5's K = 128 trailing
# update: several launches each (the small side products share the kernels); the summaries take
# the longest one
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tc_tma_kernel -s 10 -c 16 \
  -o $o/ncu_tc_tma_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline \
  --no-e2e > $o/ncu_full_tc_cfg3.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:rank_update_grouped -s 20 -c 4 \
  -o $o/ncu_update_cfg5 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline \
  --no-e2e > $o/ncu_full_update_cfg5.log 2>&1
