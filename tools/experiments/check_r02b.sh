set -u
o=gpurun_out/c2; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py tests/test_gpu_ref_primitives.py tests/test_gpu_drivers.py -m gpu -x -q > $o/gputest.log 2>&1; tail -3 $o/gputest.log
timeout 600 python tools/select_wide_bench.py $o/select_wide.jsonl > $o/select_wide.log 2>&1
timeout 600 tools/tc_sweep trq_G_cfg4 > $o/tc_sweep_m32.jsonl 2>&1
timeout 600 python tools/qr_vs_cusolver.py $o/qr_vs_cusolver.jsonl > $o/qr.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $o/bench_cfg5.json 2> $o/bench_cfg5.err
