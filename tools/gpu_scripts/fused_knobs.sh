#!/bin/bash
# fused sweep (VK_FUSED=1) timing for several VK_NVCC_FLAGS builds, cfg2
for f in "$@"; do
  VK_NVCC_FLAGS="$f" python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
  echo "[$f] $(VK_PROBE_NOCHECK=1 VK_FUSED=1 timeout 300 python tools/fused_probe.py cfg2 2>&1 | grep -E 'False|sweep' | tr '\n' ' ')"
done
python -m paper_2409_14222_b200.build --force > /dev/null 2>&1
