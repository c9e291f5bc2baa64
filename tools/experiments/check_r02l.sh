set -u
o=gpurun_out/c12; mkdir -p $o
for v in 150 175 200 230; do
  RQ_OPTIONS="sel_balance=$v" timeout 900 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $o/bench_cfg5_sb$v.json 2> $o/bench_cfg5_sb$v.err
done
