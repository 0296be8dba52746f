#!/bin/bash
# K4a solve time for several VK_NVCC_FLAGS builds on the configs in $NAMES (default cfg2)
NAMES=${NAMES:-cfg2}
i=0
for f in "$@"; do
  VK_NVCC_FLAGS="$f" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
  for rep in 1 2; do
    timeout 300 python tools/bench_kernels.py $NAMES --reps 30 --json gpurun_out/sk_$i.json > gpurun_out/sk_$i.log 2>&1
    echo "variant $i rep $rep [$f] $(python -c "
import json;d=json.load(open('gpurun_out/sk_$i.json'))
print(' '.join('%s %.4f(%.3f) acc %.4f'%(k,v['solve_ms'],v['solve_frac'],v['accumulate_ms']) for k,v in d.items()))")"
  done
  i=$((i+1))
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
