#!/bin/bash
# halves_inner (b = 128 inner product overlapped with the two-half panel),
# ssrqrcp k > 256, new gemm / rank-update shapes; cfg5 bench on/off.
o=gpurun_out/m; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_drivers.py tests/test_gpu_kernels.py -m gpu -x -q > $o/tests.log 2>&1; tail -3 $o/tests.log
for v in 1 0; do
  RQ_OPTIONS="halves_inner=$v" timeout 600 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg5_hi$v.json 2> $o/cfg5_hi$v.err
  tail -c 300 $o/cfg5_hi$v.json
done
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k cfg5 > $o/full5.log 2>&1; tail -2 $o/full5.log
