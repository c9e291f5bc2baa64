set -u
o=gpurun_out/c4; mkdir -p $o
timeout 300 python tools/panel_fast_phases.py > $o/panel_phases.log 2>&1
for v in 1024 2048 3072; do
  RQ_OPTIONS="select_cluster_max_cols=$v" timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $o/bench_cfg2_cl$v.json 2> $o/bench_cfg2_cl$v.err
done
