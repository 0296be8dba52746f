#!/bin/bash
# ncu --set full of the three K3 kernel families on their headline classes
# (re-factorisation launches): warp kernel (cfg2, s = 39), rows-in-lanes
# (cfg5, s = 74), blocked DMMA (cfg3, s = 123)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_warp -s 3 -c 1 \
  -o gpurun_out/k3_warp_cfg2 python tools/factor_probe.py cfg2 --reps 1 > gpurun_out/ncu_k3_warp.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_rows -s 3 -c 1 \
  -o gpurun_out/k3_rows_cfg5 python tools/factor_probe.py cfg5 --reps 1 > gpurun_out/ncu_k3_rows.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_blk -s 3 -c 1 \
  -o gpurun_out/k3_blk_cfg3 python tools/factor_probe.py cfg3 --reps 1 > gpurun_out/ncu_k3_blk.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:extract_blocks -s 1 -c 1 \
  -o gpurun_out/k2_extract_cfg3 python tools/factor_probe.py cfg3 --reps 1 > gpurun_out/ncu_k2.log 2>&1
# small text summaries (the reports themselves exceed what gpurun brings back)
for r in k3_warp_cfg2 k3_rows_cfg5 k3_blk_cfg3 k2_extract_cfg3; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
  rm -f gpurun_out/$r.ncu-rep
done
