#!/bin/bash
o=gpurun_out/s; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_drivers.py -m gpu -x -q > $o/tests.log 2>&1; tail -3 $o/tests.log
for v in 1 1; do
  timeout 900 python bench.py --config cfg2 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg2_f$v.json 2> $o/cfg2_f$v.err
  python -c "import json;d=json.loads(open('$o/cfg2_f$v.json').read().strip().splitlines()[-1]);print('cfg2',d['ms_per_step'],{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()})"
done
TRACE_DUMP=$o/trace_cfg2.json timeout 300 python tools/launch_trace.py cfg2 > $o/trace_cfg2.log 2>&1; tail -2 $o/trace_cfg2.log
timeout 900 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/cfg1.json 2> $o/cfg1.err
python -c "import json;d=json.loads(open('$o/cfg1.json').read().strip().splitlines()[-1]);print('cfg1',d['ms_per_step'],{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()})"
