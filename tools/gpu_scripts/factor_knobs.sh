#!/bin/bash
# factor_probe for several VK_NVCC_FLAGS builds on $NAMES (default cfg2)
NAMES=${NAMES:-cfg2}
i=0
for f in "$@"; do
  VK_NVCC_FLAGS="$f" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
  echo "variant $i [$f]"
  timeout 300 python tools/factor_probe.py $NAMES --reps 5 2>&1 | cut -c1-200
  i=$((i+1))
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
