#!/bin/bash
# ncu --set full of one panel-blocked factor class (args: TR RA CFG OUT)
TR=${1:-16}; RA=${2:-8}; CFG=${3:-cfg3}; OUT=${4:-gpurun_out/fblk}
python tools/bench_kernels.py $CFG --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:factor_blk_kernel<\(int\)$TR, \(int\)$TR, \(int\)$RA," -c 1 -o $OUT \
  python tools/bench_kernels.py $CFG --reps 1 > ${OUT}.log 2>&1
echo ncu_rc=$?
