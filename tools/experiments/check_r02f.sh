set -u
o=gpurun_out/c6; mkdir -p $o
for v in 145 200 260 340; do
  RQ_OPTIONS="sel_balance=$v" timeout 900 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $o/bench_cfg5_sb$v.json 2> $o/bench_cfg5_sb$v.err
done
