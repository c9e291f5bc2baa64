#!/bin/bash
# cfg5: select/update SM balance after this round's changes
o=gpurun_out/v; mkdir -p $o; : > $o/summary2.txt
run() { # name config opts steps
  RQ_OPTIONS="$3" timeout 900 python bench.py --config $2 --steps $4 --warmup 3 --no-cpu-baseline --no-e2e > $o/$1.json 2> $o/$1.err
  python -c "import json;d=json.loads(open('$o/$1.json').read().strip().splitlines()[-1]);print(json.dumps({'run':'$1','opts':'$3','ms_per_step':round(d['ms_per_step'],3),'kernels':{k:round(x['ms_per_step'],2) for k,x in d['kernels'].items()}}))" >> $o/summary2.txt 2>&1
}
for v in 110 130 150 170 185 200; do run cfg5_sb$v cfg5 "sel_balance=$v" 3; done
cat $o/summary2.txt
