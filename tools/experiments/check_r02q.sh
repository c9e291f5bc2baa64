#!/bin/bash
# fast panel smem row stride (fast_panel_pad 1/4/8): phases, bitwise test, cfg2
o=gpurun_out/q; mkdir -p $o; : > $o/summary.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "fast_panel" > $o/tests.log 2>&1; tail -2 $o/tests.log
PADS=1,4,8 timeout 300 python tools/panel_fast_phases.py > $o/phases.log 2>&1
for pad in 1 4 8 1 4 8; do
  RQ_OPTIONS="fast_panel_pad=$pad" timeout 600 python bench.py --config cfg2 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg2_pad$pad.json 2> $o/cfg2_pad$pad.err
  python -c "import json;d=json.loads(open('$o/cfg2_pad$pad.json').read().strip().splitlines()[-1]);print('pad$pad',d['ms_per_step'],{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()})" >> $o/summary.txt 2>&1
done
cat $o/summary.txt
