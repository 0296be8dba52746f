#!/bin/bash
# K4a build variants on one config: args = CFG then "FLAGS" strings
CFG=$1; shift
i=0
for f in "$@"; do
  VK_NVCC_FLAGS="$f" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1 && \
  python tools/bench_kernels.py $CFG --reps 30 --json gpurun_out/var_$i.json > /dev/null 2>&1
  echo "var $i [$f] rc=$? $(python -c "import json;d=json.load(open('gpurun_out/var_$i.json'));v=d['$CFG'];print(round(v['solve_ms'],4), round(v['solve_frac'],3))")"
  i=$((i+1))
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
