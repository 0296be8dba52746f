#!/bin/bash
# ncu --set full of one register-tiled factor class (arg: TR RA), cfg arg 3
TR=${1:-16}; RA=${2:-8}; CFG=${3:-cfg3}; OUT=${4:-gpurun_out/ftile}
python tools/bench_kernels.py $CFG --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:factor_tile_kernel<\(int\)$TR, \(int\)$TR, \(int\)$RA," -c 1 -o $OUT \
  python tools/bench_kernels.py $CFG --reps 1 > ${OUT}.log 2>&1
echo ncu_rc=$?
