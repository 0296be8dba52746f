#!/bin/bash
# bench.py sweep step time for several VK_NVCC_FLAGS builds (no CPU leg)
i=0
for f in "$@"; do
  VK_NVCC_FLAGS="$f" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
  for rep in 1 2; do
    timeout 300 python bench.py --no-cpu --steps 50 > gpurun_out/bn_$i.log 2>&1
    echo "variant $i rep $rep [$f] $(tail -1 gpurun_out/bn_$i.log | python -c "
import json,sys;d=json.loads(sys.stdin.read())
print('step %.4f ms value %.4e solve %.4f acc %.4f e2e %.4e tts %.2f' % (d['ms_per_step'], d['value'], d['sweep']['ms_solve'], d['sweep']['ms_accumulate'], d['e2e']['value'], d['mg_fgmres']['tts_ms_median']))")"
  done
  i=$((i+1))
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
