#!/bin/bash
# Round measurement bundle (1 GPU): bench line, TTS, launch list, ncu of K4a.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/m_bench.log 2>&1; echo bench_rc=$?
python tools/bench_kernels.py --tts --json gpurun_out/m_tts.json > gpurun_out/m_tts.log 2>&1; echo tts_rc=$?
python bench.py --steps 2 --warmup 1 > gpurun_out/m_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/m_ncu_launch.log 2>&1
echo launch_rc=$?
ncu --set full --clock-control none --import-source on -k regex:patch_solve -s 3 -c 1 \
    -o gpurun_out/m_sweep python bench.py --steps 2 --warmup 1 > gpurun_out/m_ncu_full.log 2>&1
echo ncu_full_rc=$?
