#!/bin/bash
# ncu --set full of one look-ahead factor class (args: RA TC CFG OUT)
RA=${1:-4}; TC=${2:-7}; CB=${5:-19}; CFG=${3:-cfg3}; OUT=${4:-gpurun_out/fla}
python tools/bench_kernels.py $CFG --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:factor_la_kernel<\(int\)$RA, \(int\)$TC, \(int\)$CB>" -c 1 -o $OUT \
  python tools/bench_kernels.py $CFG --reps 1 > ${OUT}.log 2>&1
echo ncu_rc=$?
