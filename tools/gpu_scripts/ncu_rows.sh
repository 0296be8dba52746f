mkdir -p gpurun_out
VK_FACTOR_TIMING=1 timeout 300 python tools/factor_probe.py cfg2 cfg3 cfg4 cfg5 --reps 2 > gpurun_out/factor3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_rows -s 3 -c 1 -o gpurun_out/rows_cfg2 python tools/factor_probe.py cfg2 --reps 1 > gpurun_out/ncu_rows_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_rows -s 9 -c 3 -o gpurun_out/rows_cfg3 python tools/factor_probe.py cfg3 --reps 1 > gpurun_out/ncu_rows_cfg3.log 2>&1
