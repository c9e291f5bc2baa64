#!/bin/bash
# Round-end refresh: GPU tests, bench lines for every config, reference arm,
# and the ncu launch list of the cfg2 bench command.  Outputs in gpurun_out/g.
set -u
o=gpurun_out/g; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c > $o/bench_$c.json 2> $o/bench_$c.err
done
timeout 300 python bench.py --impl reference > $o/bench_ref_cfg2.json 2> $o/bench_ref_cfg2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include timed/ \
  --csv --log-file $o/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e > $o/ncu_launch.log 2>&1
tail -c 300 $o/bench_*.json
# parity at full size (cfg1-cfg4, the cfg5 recipe at 8192^2) and the sweep
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python tools/full_parity.py $c $o/parity_$c.json > /dev/null 2>&1
done
timeout 900 python tools/full_parity.py cfg5 $o/parity_cfg5_8192.json m=8192 n=8192 > /dev/null 2>&1
timeout 1500 python tools/parity_sweep.py $o/parity_sweep.jsonl > /dev/null 2>&1
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/g/parity_cfg*.json")):
    d = json.load(open(f))
    print(f, d.get("pivots_identical"), d.get("R_rel_err"), d.get("sigma_max_rel_err"))
rows = [json.loads(l) for l in open("gpurun_out/g/parity_sweep.jsonl")]
print("sweep", len(rows), "ok", sum(r.get("ok", False) for r in rows))
PY
