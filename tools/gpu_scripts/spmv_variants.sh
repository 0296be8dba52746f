#!/bin/bash
# residual SpMV for several stream-block shapes: args = "THREADS U" pairs
for c in "$@"; do
  set -- $c
  VK_NVCC_FLAGS="-DVK_STREAM_THREADS=$1 -DVK_STREAM_U=$2" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1 && \
  timeout 300 python tools/bench_kernels.py --reps 20 --json gpurun_out/sv.json > /dev/null 2>&1
  echo "shape $1x$2 rc=$? $(python -c "
import json;d=json.load(open('gpurun_out/sv.json'))
print(' '.join('%s %.4f(%.3f)'%(k,v['residual_ms'],v['residual_frac']) for k,v in d.items()))")"
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
