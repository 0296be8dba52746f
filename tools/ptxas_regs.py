#!/usr/bin/env python
"""Registers / spills per kernel from `nvcc -Xptxas -v` output on stdin."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        d = re.search(r"(\w+_kernel)(I\w*?E)?E", name)
        cur = name
        short = re.sub(r"_ZN\w*?_GLOBAL__N__\w+?\d+", "", name)
        cur = short[:70]
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        spill = m.group(1)
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:70s} regs {m.group(1):>4s} spill {spill}")
        cur = None
