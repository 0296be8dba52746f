#!/bin/bash
# transfer_probe (residual / prolong / restrict) for several VK_NVCC_FLAGS builds,
# CUDA-event medians plus ncu per-launch durations (cold, clean L2) for cfg2
i=0
for f in "$@"; do
  VK_NVCC_FLAGS="$f" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1 && \
  timeout 300 python tools/transfer_probe.py --reps 30 --json gpurun_out/cv_$i.json > gpurun_out/cv_$i.log 2>&1
  echo "variant $i [$f] rc=$?"
  python -c "
import json;d=json.load(open('gpurun_out/cv_$i.json'))
for k,v in d.items(): print(' ', k, ' '.join('%s %.1f/%.1fus(%.2f)'%(o, v[o+'_cold_us'], v[o+'_warm_us'], v[o+'_cold_frac']) for o in ('residual','prolong','restrict','copy')))"
  timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum --csv -k regex:csr_ python tools/transfer_probe.py cfg2 cfg5 --reps 2 2>/dev/null \
    | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10 and r[0].isdigit()]
d=collections.defaultdict(list)
for r in rows: d[r[8]].append(float(r[-1]))
print('  ncu us by grid:', {k: round(min(v),2) for k,v in d.items()})"
  i=$((i+1))
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
