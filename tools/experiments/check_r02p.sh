#!/bin/bash
# cfg2: panel / inner-product SM split (overlap_panel_ctas); cfg5: select / update split (sel_balance)
o=gpurun_out/p; mkdir -p $o; : > $o/summary.txt
run() {  # tag config steps options
  RQ_OPTIONS="$4" timeout 600 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e > $o/$1.json 2> $o/$1.err
  python -c "import json;d=json.loads(open('$o/$1.json').read().strip().splitlines()[-1]);print('$1','$4',d['ms_per_step'],d.get('steps_ms'),{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()})" >> $o/summary.txt 2>&1
}
for q in 0 48 64 80 100 0; do run cfg2_q$q cfg2 8 "overlap_panel_ctas=$q"; done
for sb in 230 200 260 300; do run cfg5_sb$sb cfg5 2 "sel_balance=$sb"; done
cat $o/summary.txt
