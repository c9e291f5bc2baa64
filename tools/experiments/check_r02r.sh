#!/bin/bash
# re-entry baseline: full gpu suite, cfg2 bench, cfg2/cfg5 trace dumps
o=gpurun_out/r; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/tests.log 2>&1; tail -3 $o/tests.log
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 > $o/cfg2.json 2> $o/cfg2.err; tail -c 600 $o/cfg2.json
TRACE_DUMP=$o/trace_cfg2.json timeout 300 python tools/launch_trace.py cfg2 > $o/trace_cfg2.log 2>&1; tail -3 $o/trace_cfg2.log
TRACE_DUMP=$o/trace_cfg5.json timeout 300 python tools/launch_trace.py cfg5 > $o/trace_cfg5.log 2>&1; tail -3 $o/trace_cfg5.log
