#!/bin/bash
# end-of-round check: full GPU suite, smoke, default bench + reference arm
o=gpurun_out/final; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/gputest.log 2>&1; tail -2 $o/gputest.log
timeout 300 python __graft_entry__.py smoke > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; tail -c 300 $o/bench_default.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err; tail -c 200 $o/bench_ref.json; echo
for c in cfg2 cfg5; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err
python -c "import json;d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]);print('$c',d['ms_per_step'],{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()})"
done
