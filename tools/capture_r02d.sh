o=gpurun_out/r2d; mkdir -p $o
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tc_tma_kernel -s 10 -c 16 \
  -f -o $o/ncu_tc_tma_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline \
  --no-e2e > $o/ncu_full_tc_cfg3.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:rank_update_grouped -s 20 -c 4 \
  -f -o $o/ncu_update_cfg5 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline \
  --no-e2e > $o/ncu_full_update_cfg5.log 2>&1
ls -la $o/*.ncu-rep
