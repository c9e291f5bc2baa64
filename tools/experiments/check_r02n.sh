#!/bin/bash
# grouped trailing update: C-tile TMA prefetch variants (ru_tma 1/2/3)
o=gpurun_out/n; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "rank_update" > $o/tests.log 2>&1; tail -2 $o/tests.log
timeout 600 python tools/tc_bench.py --only ru_b64_cfg2,ru_b64_half,ru_b128_mid,qrb_update > $o/tc.jsonl 2> $o/tc.err
for v in 1 2 3; do
  RQ_OPTIONS="ru_tma=$v" timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg2_ru$v.json 2> $o/cfg2_ru$v.err
done
for v in 1 2 3; do
  RQ_OPTIONS="ru_tma=$v" timeout 600 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg5_ru$v.json 2> $o/cfg5_ru$v.err
done
timeout 900 python -m pytest tests/test_gpu_drivers.py -m gpu -x -q > $o/drivers.log 2>&1; tail -2 $o/drivers.log
