#!/usr/bin/env python
"""Summarise VK_FACTOR_TIMING logs (tools/gpu_scripts/ftime.sh): per config the
re-factor time and the large size classes (second, warm factorization)."""
import re
import sys

seen = {}
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ftime.log"):
    m = re.match(r"\[vk_factor\] class <=(\d+): (\d+) patches, ([0-9.]+) ms", line)
    if m:
        seen[(m.group(1), m.group(2))] = m.group(3)
    if line.startswith("cfg"):
        fs = re.search(r'"factor_s": ([0-9.]+)', line).group(1)
        print(line[:4], "factor_s", fs, {k[0]: (k[1], v) for k, v in seen.items() if int(k[1]) > 400})
        seen = {}
