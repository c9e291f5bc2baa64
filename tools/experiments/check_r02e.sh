set -u
o=gpurun_out/c5; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k select > $o/gputest.log 2>&1; tail -2 $o/gputest.log
timeout 600 python tools/select_wide_bench.py $o/select_wide.jsonl > $o/select_wide.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $o/bench_cfg5.json 2> $o/bench_cfg5.err
