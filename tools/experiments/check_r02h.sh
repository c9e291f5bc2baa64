set -u
o=gpurun_out/c8; mkdir -p $o
RQ_LIB_PATH=altlib/librqrcp_ref.so timeout 300 python tools/panel_fast_dump.py $o/panel_ref.npz > $o/dump_ref.log 2>&1
timeout 300 python tools/panel_fast_dump.py $o/panel_new.npz --compare $o/panel_ref.npz > $o/dump_cmp.log 2>&1; tail -3 $o/dump_cmp.log
timeout 300 python tools/panel_fast_phases.py > $o/panel_phases.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_drivers.py -m gpu -x -q > $o/gputest.log 2>&1; tail -2 $o/gputest.log
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $o/bench_cfg2.json 2> $o/bench_cfg2.err
