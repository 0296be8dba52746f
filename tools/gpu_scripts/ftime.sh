#!/bin/bash
# per-class factor timings for all configs -> $1 (default gpurun_out/ftime.log)
OUT=${1:-gpurun_out/ftime.log}
VK_FACTOR_TIMING=1 python tools/bench_kernels.py cfg2 cfg3 cfg4 cfg5 --reps 2 > $OUT 2>&1
echo ftime_rc=$?
