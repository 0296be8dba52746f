#!/bin/bash
# bench_kernels for several VK_NVCC_FLAGS builds: args = "FLAGS" strings
i=0
for f in "$@"; do
  VK_NVCC_FLAGS="$f" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1 && \
  timeout 300 python tools/bench_kernels.py --reps 20 --json gpurun_out/bv_$i.json > /dev/null 2>&1
  echo "variant $i [$f] rc=$? $(python -c "
import json;d=json.load(open('gpurun_out/bv_$i.json'))
print(' '.join('%s %.4f(%.3f)'%(k,v['solve_ms'],v['solve_frac']) for k,v in d.items()))")"
  i=$((i+1))
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
