#!/bin/bash
o=gpurun_out/s; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "panel" > $o/tests.log 2>&1; tail -3 $o/tests.log
timeout 300 python tools/panel_driver_phases.py > $o/panel_driver_phases.log 2>&1; cat $o/panel_driver_phases.log | tail -12
timeout 900 python -m pytest tests/test_gpu_drivers.py -m gpu -x -q > $o/tests2.log 2>&1; tail -3 $o/tests2.log
for i in 1 2; do
  timeout 600 python bench.py --config cfg2 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg2.json 2> $o/cfg2.err
  python -c "import json;d=json.loads(open('$o/cfg2.json').read().strip().splitlines()[-1]);print('cfg2',d['ms_per_step'],{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()})"
done
