#!/bin/bash
# fast panel: chunk loads pipelined behind the DMMA work; select: release-arrival grid barrier
o=gpurun_out/o; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_drivers.py -m gpu -x -q > $o/tests.log 2>&1; tail -2 $o/tests.log
timeout 300 python tools/panel_fast_phases.py > $o/phases.log 2>&1
for v in 0 1 0 1; do
  RQ_OPTIONS="sel_bar_release=$v,ru_tma=${RU:-2}" timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg2_rel$v.json 2> $o/cfg2_rel$v.err
  python -c "import json;d=json.loads(open('$o/cfg2_rel$v.json').read().strip().splitlines()[-1]);print('rel$v',d['ms_per_step'],{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()})" >> $o/summary.txt
done
cat $o/summary.txt
