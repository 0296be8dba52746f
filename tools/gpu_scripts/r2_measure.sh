#!/bin/bash
# Round-2 measurement bundle (1 GPU): bench line, launch list of the timed
# region, ncu --set full of the headline K4a launch (cfg3 chunk kernel).
set -u
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --headline-only --no-cpu > gpurun_out/r2_plain.log 2>&1
echo plain_rc=$?
VK_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 1 --headline-only --no-cpu > gpurun_out/r2_ncu_launch.log 2>&1
echo launch_rc=$?
VK_PROFILE_TIMED=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:patch_solve -c 1 -o gpurun_out/r2_sweep_cfg3 \
    python bench.py --steps 2 --warmup 1 --headline-only --no-cpu > gpurun_out/r2_ncu_full.log 2>&1
echo ncu_full_rc=$?
